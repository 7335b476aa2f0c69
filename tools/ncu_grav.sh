# Full ncu captures (one launch each) of the gravity kernels and the stage
# kernel on C3, for profiles/: bash tools/ncu_grav.sh [tag] [kernel regex...]
tag=${1:-r02}; shift
mkdir -p gpurun_out
kernels=${@:-amr_l2p_kernel amr_wx_kernel amr_m2l_fused_kernel amr_m2m_kernel amr_m2l_mono_kernel stage_kernel}
for k in $kernels; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 6 -c 1 -f \
    -o gpurun_out/${tag}_$k python tools/grav_amr_bench.py 2 5 3 > gpurun_out/${tag}_ncu_$k.log 2>&1
  echo "$k rc=$?"
done
