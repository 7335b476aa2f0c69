mkdir -p gpurun_out
for k in amr_l2p_kernel amr_wx_kernel amr_m2l_fused_kernel amr_m2m_kernel amr_m2l_mono_kernel; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 6 -c 1 -f -o gpurun_out/r02b_$k python tools/grav_amr_bench.py 2 5 3 > gpurun_out/r02b_ncu_$k.log 2>&1
  echo "$k rc=$?"
done
