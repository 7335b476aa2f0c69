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
