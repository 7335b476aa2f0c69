"""HostStepPipeline (host-buffer stepping with overlapped copies) gives, step
for step, the bytes of the plain set_interior -> step -> get_interior path."""
import numpy as np
import pytest

from paper_2412_15518_b200 import amr
from paper_2412_15518_b200.driver import GravityHydroDriver, HostStepPipeline, HydroDriver

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("gravity", [False, True])
def test_pipeline_equals_sequential(gravity):
    import torch

    Drv = GravityHydroDriver if gravity else HydroDriver

    def fresh():  # same construction -> same ghost history (ghost.hpp:10-13)
        f = amr.build_scenario(amr.Scenario.rotating_star, 1, 3)
        f.alloc()
        return f, Drv(f)

    f, drv = fresh()
    s0 = f.scenario_state(amr.Scenario.rotating_star)
    # reference: independent inputs, one plain step each
    rng = np.random.default_rng(3)
    inputs = [s0 * (1.0 + 1e-3 * rng.uniform(-1, 1, s0.shape)) for _ in range(4)]
    want = []
    for x in inputs:
        f.set_interior(x)
        drv.step()
        want.append(f.get_interior())
    if gravity:
        drv.close()
    f, drv = fresh()
    pins = [torch.from_numpy(x).pin_memory() for x in inputs]
    outs = [torch.empty_like(p).pin_memory() for p in pins]
    pipe = HostStepPipeline(drv)
    for p, o in zip(pins, outs):
        pipe.step(p, o)
    pipe.synchronize()
    for o, w in zip(outs, want):
        assert o.numpy().tobytes() == w.tobytes()
    if gravity:
        drv.close()


@pytest.mark.parametrize("case", ["hydro", "hydro_dt", "reflux", "grav1", "grav3", "grav6", "exact3"])
def test_step_io_equals_set_step_get(case):
    """tmgpu_forest_step_io (input scattered in the step's first pass, output
    written by the last stage's epilogue) == set_interior + step + get_interior,
    bit for bit, incl. the late-correction cases (reflux, 6-solve cadence) that
    gather after the loop and the fixed-dt path without the fused scatter."""
    import torch

    def make():
        f = amr.build_scenario(amr.Scenario.rotating_star, 1, 3)
        f.alloc()
        kw = {"exact_ghosts": case == "exact3"}
        if case.startswith("grav") or case == "exact3":
            d = GravityHydroDriver(f, solves_per_step=int(case[-1]), **kw)
        else:
            d = HydroDriver(f, reflux=case == "reflux")
        return f, d

    dt = 1e-3 if case == "hydro_dt" else None
    s0 = amr.build_scenario(amr.Scenario.rotating_star, 1, 3).scenario_state(amr.Scenario.rotating_star)
    f, d = make()
    want = []
    for k in range(3):
        x = s0 * (1.0 + 1e-4 * k)
        f.set_interior(x)
        d.step(dt=dt)
        want.append(f.get_interior())
    g, e = make()
    for k in range(3):
        x = torch.from_numpy(s0 * (1.0 + 1e-4 * k)).cuda()
        out = torch.empty_like(x)
        e.step(dt=dt, io=(x, out))
        assert out.cpu().numpy().tobytes() == want[k].tobytes(), f"step {k}"
        assert g.get_interior().tobytes() == want[k].tobytes()
