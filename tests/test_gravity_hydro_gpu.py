"""The gravity + hydro step (GravityHydroDriver) vs the oracle composition
(tests/helpers.py oracle_gravity_step): AMR FMM specification
(gravity_amr_oracle.c, with the angular-momentum correction) at 1, 3 or 6
solves per step -> per RK stage: ghost fill (tmo_fill_ghosts_sync) -> stage
with the gravity source (tmo_stage_subgrid_grav) -> rk3_combine. Bitwise."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2412_15518_b200 import amr
from paper_2412_15518_b200.driver import GravityHydroDriver
from paper_2412_15518_b200.gravity import forest_leaf_array

from helpers import interior_to_ghosted, oracle_gravity_step

pytestmark = pytest.mark.gpu



@pytest.mark.parametrize("cadence", [1, 3, 6])
@pytest.mark.parametrize("exact", [False, True])
def test_gravity_hydro_step_bitwise_vs_oracle(exact, cadence):
    if exact and cadence == 6:
        pytest.skip("the 6-solve cadence runs on the fused (ping-pong) step only")
    f = amr.build_scenario(amr.Scenario.rotating_star, 1, 3)
    st = f.scenario_state(amr.Scenario.rotating_star)
    f.alloc()
    f.set_interior(st)
    lv = forest_leaf_array(f)
    o = O.Oracle()
    t = o.tree([int(p) for p in f.leaves()])
    grids = [np.ascontiguousarray(g) for g in interior_to_ghosted(st)]
    drv = GravityHydroDriver(f, am=True, exact_ghosts=exact, solves_per_step=cadence)
    dt = 2e-3
    for step in range(2):
        drv.step(dt=dt)
        grids = oracle_gravity_step(o, t, grids, lv, dt, cadence)
        got = f.get_interior()
        want = np.stack([g.reshape(5, 12, 12, 12)[:, 2:10, 2:10, 2:10].reshape(5, 512) for g in grids])
        assert got.tobytes() == want.tobytes(), f"step {step}"
    drv.close()


def test_gravity_cadences_differ_and_converge():
    """The three cadences are different schemes (not relabellings) and agree
    to O(dt^2) relative: per-stage fields differ from the held field."""
    res = {}
    for cad in (1, 3, 6):
        f = amr.build_scenario(amr.Scenario.rotating_star, 2, 3)
        st = f.scenario_state(amr.Scenario.rotating_star)
        f.alloc()
        f.set_interior(st)
        drv = GravityHydroDriver(f, am=True, solves_per_step=cad)
        for _ in range(2):
            drv.step(dt=2e-3)
        res[cad] = f.get_interior()
        drv.close()
    m1, m3, m6 = (res[c][:, 1:4] for c in (1, 3, 6))
    scale = np.abs(m3).max()
    assert np.abs(m1 - m3).max() > 0 and np.abs(m3 - m6).max() > 0
    assert np.abs(m1 - m3).max() < 1e-2 * scale and np.abs(m3 - m6).max() < 1e-2 * scale


def test_gravity_cadence_rejects_bad_arguments():
    f = amr.build_scenario(amr.Scenario.rotating_star, 1, 2)
    f.alloc()
    with pytest.raises(ValueError):
        GravityHydroDriver(f, solves_per_step=2)
    drv = GravityHydroDriver(f, solves_per_step=6, exact_ghosts=True)
    with pytest.raises(Exception, match="6-solve"):
        drv.step(dt=1e-3)
    drv.close()


def test_gravity_source_pulls_momentum_inward():
    """Sanity of the coupling: with minus without gravity, one step adds
    momentum toward the star centre inside the star."""
    from paper_2412_15518_b200.driver import HydroDriver

    outs = []
    for grav in (True, False):
        f = amr.build_scenario(amr.Scenario.rotating_star, 2, 3)
        st = f.scenario_state(amr.Scenario.rotating_star)
        f.alloc()
        f.set_interior(st)
        drv = GravityHydroDriver(f, am=True) if grav else HydroDriver(f)
        drv.step(dt=1e-3)
        outs.append(f.get_interior())
    d = outs[0] - outs[1]
    x = O.leaf_centres(forest_leaf_array(f)).reshape(-1, 512, 3)
    rad = (np.stack([d[:, 1], d[:, 2], d[:, 3]], -1) * (x - 0.5)).sum(-1)
    dense = st[:, 0] > 0.3
    assert (rad[dense] < 0).mean() > 0.95



@pytest.mark.parametrize("cadence", [0, 3, 6])
def test_step_graph_replay_equals_direct(cadence):
    """The one-GPU step replayed as a cached CUDA graph (the default after the
    first step) equals the directly enqueued step bit for bit, over CFL steps,
    alternating device output buffers (several cached graphs) and a setter
    that drops the cache (reflux on) mid-run."""
    import ctypes as C

    import torch

    from paper_2412_15518_b200 import _lib
    from paper_2412_15518_b200.driver import HydroDriver, lib

    runs = []
    for graph in (True, False):
        f = amr.build_scenario(amr.Scenario.rotating_star, 1, 3)
        f.alloc()
        f.set_interior(f.scenario_state(amr.Scenario.rotating_star))
        drv = GravityHydroDriver(f, am=True, solves_per_step=cadence) if cadence else HydroDriver(f)
        drv.graph = graph
        n = f.leaf_count() * 5 * 512
        bufs = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
        outs = []
        for k in range(6):
            if k == 4:  # a setter mid-run: the cached graphs must be dropped
                err = _lib.TmgpuError()
                _lib.check(lib.tmgpu_forest_set_reflux(f.h, 1, C.byref(err)), err)
            if k in (2, 3):  # output through alternating device buffers
                drv.step(io=(None, bufs[k % 2]))
                outs.append(bufs[k % 2].cpu().numpy().tobytes())
            else:
                drv.step()
            outs.append(f.get_interior().tobytes())
        runs.append(outs)
    assert runs[0] == runs[1]
