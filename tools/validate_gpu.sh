#!/bin/bash
# Round-end GPU validation on 4 GPUs: gpu tests, smoke, bench N=1/2/4 and configs[4] at N=4 (logs into gpurun_out/).
export PYTHONUNBUFFERED=1
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port"
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/v_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/v_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > gpurun_out/v_smoke.log 2>&1; tail -1 gpurun_out/v_smoke.log
timeout 600 python bench.py > gpurun_out/v_n1.log 2>gpurun_out/v_n1.err; echo "n1 rc $?"
timeout 400 $T 29611 --nproc-per-node=2 bench.py --gpus 2 > gpurun_out/v_n2.log 2>gpurun_out/v_n2.err; echo "n2 rc $?"
timeout 400 $T 29612 --nproc-per-node=4 bench.py --gpus 4 > gpurun_out/v_n4.log 2>gpurun_out/v_n4.err; echo "n4 rc $?"
timeout 400 $T 29613 --nproc-per-node=4 bench.py --gpus 4 --scenario dwd --max-level 7 --steps 10 --warmup 3 > gpurun_out/v_c5_n4.log 2>gpurun_out/v_c5_n4.err; echo "c5 rc $?"
for f in v_n1 v_n2 v_n4 v_c5_n4; do tail -1 gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d.get('clocks'))"; done
