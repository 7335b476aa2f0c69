"""Where the e2e step's time goes on one GPU (C3 gravity+hydro): device-only
steps; steps + interior scatter/gather on the device; the full HostStepPipeline;
the pipeline's copies alone. CUDA events, 30 steps each."""
import numpy as np
import torch

from paper_2412_15518_b200 import amr
from paper_2412_15518_b200.driver import GravityHydroDriver, HostStepPipeline

f = amr.build_scenario(amr.Scenario.rotating_star, 2, 5, 0.1)
state = f.scenario_state(amr.Scenario.rotating_star)
f.alloc()
f.set_interior(state)
drv = GravityHydroDriver(f)
cs = torch.cuda.current_stream()
K = 30


def timed(fn, stream=None):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream or cs)
    for _ in range(K):
        fn()
    b.record(stream or cs)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K


dev = torch.from_numpy(state).cuda()
out = torch.empty_like(dev)
print("step only      %.3f ms" % timed(lambda: drv.step(stream=cs.cuda_stream, sync=False)))


def with_io():
    f.set_interior(dev, stream=cs.cuda_stream, sync=False)
    drv.step(stream=cs.cuda_stream, sync=False)
    f.get_interior(out, stream=cs.cuda_stream, sync=False)


print("step + dev I/O %.3f ms" % timed(with_io))
print("step_io        %.3f ms" % timed(lambda: drv.step(stream=cs.cuda_stream, sync=False, io=(dev, out))))
pin_in = torch.from_numpy(np.ascontiguousarray(state)).pin_memory()
pin_out = torch.empty_like(pin_in).pin_memory()
pipe = HostStepPipeline(drv)
print("pipeline       %.3f ms" % timed(lambda: pipe.step(pin_in, pin_out), pipe.h2d))
K = 100
print("pipeline x100  %.3f ms" % timed(lambda: pipe.step(pin_in, pin_out), pipe.h2d))
K = 30
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def copies():
    with torch.cuda.stream(s1):
        dev.copy_(pin_in, non_blocking=True)
    with torch.cuda.stream(s2):
        pin_out.copy_(out, non_blocking=True)
    cs.wait_stream(s1)
    cs.wait_stream(s2)


print("copies only    %.3f ms" % timed(copies))


def step_and_copies():
    with torch.cuda.stream(s1):
        dev.copy_(pin_in, non_blocking=True)
    with torch.cuda.stream(s2):
        pin_out.copy_(out, non_blocking=True)
    drv.step(stream=cs.cuda_stream, sync=False)
    cs.wait_stream(s1)
    cs.wait_stream(s2)


print("step || copies %.3f ms" % timed(step_and_copies))
drv.close()
