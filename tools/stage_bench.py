"""Quick kernel-level measurement of the aggregated stage (slice contract,
device-resident slices). Not the driver bench (bench.py); used for ncu runs."""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_15518_b200 import _lib, hydro  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--count", type=int, default=5888)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--quick", action="store_true")
ap.add_argument("--fast", action="store_true")
a = ap.parse_args()
if a.quick:
    a.iters = 3

g = hydro.StageGeom(vars=5)
ins, outs = g.in_slice(), g.out_slice()
rng = np.random.default_rng(1)
n = 12 ** 3
one = np.zeros(ins)
hydro.encode_header(hydro.StageParams(hydro.Mode.euler, 1 / 256, 0.4 / 512), one)
rho = rng.uniform(0.2, 2.0, n); u, v, w = (rng.uniform(-.5, .5, n) for _ in range(3)); p = rng.uniform(0.2, 2, n)
one[8:] = np.concatenate([rho, rho * u, rho * v, rho * w, p / 0.4 + 0.5 * rho * (u * u + v * v + w * w)])
din = torch.from_numpy(np.tile(one, a.count)).cuda()
dout = torch.zeros(a.count * outs, dtype=torch.float64, device="cuda")
flags = _lib.TMGPU_FAST if a.fast else 0
err = _lib.TmgpuError()
st = torch.cuda.current_stream().cuda_stream


def call():
    rc = _lib.lib.tmgpu_stage_fused(din.data_ptr(), dout.data_ptr(), ins, outs, a.count, 8, 2, 5,
                                    flags, st, C.byref(err))
    _lib.check(rc, err)


for _ in range(3):
    call()
torch.cuda.synchronize()
t = []
for _ in range(a.iters):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); call(); e1.record(); torch.cuda.synchronize()
    t.append(e0.elapsed_time(e1))
ms = float(np.median(t))
cells = a.count * 512
peak = C.c_double(0); pms = C.c_double(0)
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "probes"))
import probe  # noqa: E402  tools/probes/libtmprobe.so

probe.load().tmgpu_fp64_peak(20000, C.byref(peak), C.byref(pms), None)
res = {"count": a.count, "fast": a.fast, "ms_median": ms, "ms_min": min(t),
       "cell_stage_per_s": cells / (ms * 1e-3),
       "slice_GBps": a.count * (ins + outs) * 8 / (ms * 1e-3) / 1e9,
       "alg_TFLOPs_633": cells * 633.25 / (ms * 1e-3) / 1e12,
       "fp64_peak_TFLOPs": peak.value}
print(json.dumps(res))
