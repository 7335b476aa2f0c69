"""AMR FMM gravity timing on a scenario forest (default C3: rotating star,
leaf levels 2..5) and the gravity+hydro step; for ncu runs and quick checks."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2412_15518_b200 import amr
from paper_2412_15518_b200.driver import GravityHydroDriver, HydroDriver
from paper_2412_15518_b200.gravity import GravityAMR, forest_leaf_array

lo = int(sys.argv[1]) if len(sys.argv) > 1 else 2
hi = int(sys.argv[2]) if len(sys.argv) > 2 else 5
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
f = amr.build_scenario(amr.Scenario.rotating_star, lo, hi)
f.alloc()
f.set_interior(f.scenario_state(amr.Scenario.rotating_star))
t0 = time.perf_counter()
G = GravityAMR(forest_leaf_array(f))
print("plan+upload s", round(time.perf_counter() - t0, 3), "info (levels, nodes, W/X, U)", G.info())
n = f.leaf_count() * 512
phi = torch.empty(n, dtype=torch.float64, device="cuda")
g = torch.empty(3 * n, dtype=torch.float64, device="cuda")


def timed(fn, reps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


G.mass_from_arena(f)
for am in (False, True):
    ms = timed(lambda: G.solve(None, am=am, phi=phi, g=g, sync=False), reps)
    print(f"solve am={am}: {ms:.3f} ms  ({n / ms / 1e3:.3e} cells/s)")
G.set_timing(True)
for _ in range(reps):
    G.solve(None, am=True, phi=phi, g=g, sync=False)
torch.cuda.synchronize()
tot, ns = G.timing()
G.set_timing(False)
print("phases ms/solve:", {k: round(v / ns, 4) for k, v in tot.items()})
hd = HydroDriver(f)
print(f"hydro step: {timed(lambda: hd.step(sync=False), reps):.3f} ms")
import ctypes as C  # noqa: E402
from paper_2412_15518_b200 import _lib  # noqa: E402
L = _lib.lib
L.tmgpu_forest_set_timing.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
L.tmgpu_forest_timing.argtypes = [C.c_void_p] + [C.POINTER(C.c_double)] * 3 + [C.POINTER(C.c_longlong)]
L.tmgpu_forest_set_timing(f.h, 1, None)
for _ in range(reps):
    hd.step(sync=False)
torch.cuda.synchronize()
tc, te, ts, nst = C.c_double(), C.c_double(), C.c_double(), C.c_longlong()
L.tmgpu_forest_timing(f.h, C.byref(tc), C.byref(te), C.byref(ts), C.byref(nst))
L.tmgpu_forest_set_timing(f.h, 0, None)
print(f"stage launch: {ts.value / (3 * max(nst.value, 1)):.4f} ms  exchange: {te.value / (3 * max(nst.value, 1)):.4f} ms")
for sps in (1, 3, 6):
    gd = GravityHydroDriver(f, solves_per_step=sps)
    print(f"gravity+hydro step ({sps} solves): {timed(lambda: gd.step(sync=False), reps):.3f} ms")
    gd.check()
    gd.close()
