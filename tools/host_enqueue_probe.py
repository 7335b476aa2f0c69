"""Probe: host time to enqueue one asynchronous gravity+hydro step (ctypes +
C++ launches) against its device time, on one GPU (C3 star). A step whose
enqueue time approaches its device time would be launch-bound."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_15518_b200 import amr  # noqa: E402
from paper_2412_15518_b200.driver import GravityHydroDriver, HydroDriver  # noqa: E402

for grav in (True, False):
    f = amr.build_scenario(amr.Scenario.rotating_star, 2, 5, 0.1)
    f.alloc()
    f.set_interior(f.scenario_state(amr.Scenario.rotating_star))
    drv = GravityHydroDriver(f) if grav else HydroDriver(f)
    sp = torch.cuda.current_stream().cuda_stream
    for _ in range(5):
        drv.step(stream=sp, sync=False)
    torch.cuda.synchronize()
    K = 30
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    for _ in range(K):
        drv.step(stream=sp, sync=False)
    host = (time.perf_counter() - t0) / K * 1e3
    e1.record()
    torch.cuda.synchronize()
    print(f"{'gravity+hydro' if grav else 'hydro'}: host enqueue {host:.3f} ms/step, "
          f"device {e0.elapsed_time(e1) / K:.3f} ms/step")
    drv.check(stream=sp)
