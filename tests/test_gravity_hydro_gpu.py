"""The gravity + hydro step (GravityHydroDriver) vs the oracle composition:
AMR FMM specification (gravity_amr_oracle.c, with the angular-momentum
correction) -> per RK stage: ghost fill (tmo_fill_ghosts_sync) -> stage with the
gravity source (tmo_stage_subgrid_grav) -> rk3_combine. Bitwise."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
from paper_2412_15518_b200 import amr
from paper_2412_15518_b200.driver import GravityHydroDriver
from paper_2412_15518_b200.gravity import forest_leaf_array

from helpers import interior_to_ghosted

pytestmark = pytest.mark.gpu

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)


def oracle_gravity_step(o, t, grids, lv, dt, gamma=1.4):
    n = len(grids)
    h = 1.0 / (8.0 * 2.0 ** lv[:, 0].astype(np.float64))
    interior = [g.reshape(5, 12, 12, 12)[:, 2:10, 2:10, 2:10].reshape(5, 512).copy() for g in grids]
    m = np.stack([u[0] for u in interior]) * (h * h * h)[:, None]
    _, gfield, _ = o.grav_amr(lv, m, flags=1)
    u0 = interior
    bad = (C.c_int * 3)()
    for stage in (1, 2, 3):
        t.fill_ghosts(grids)
        outs = []
        for i in range(n):
            hdr = np.array([1.0, h[i], dt, gamma, 0.0, 0.0, 0.0, 0.0])
            out = np.zeros(5 * 512 + 6 * 5 * 64 + 1)
            gi = np.ascontiguousarray(gfield[:, i * 512:(i + 1) * 512])
            rc = o.lib.tmo_stage_subgrid_grav(hdr.ctypes.data_as(dp), 8, 2, 5, grids[i].ctypes.data_as(dp),
                                              gi.ctypes.data_as(dp), out.ctypes.data_as(dp), bad)
            assert rc == 0
            v = out[:2560].reshape(5, 512)
            if stage == 2:
                v = u0[i] + 0.25 * (v - u0[i])
            elif stage == 3:
                v = u0[i] + (2.0 / 3.0) * (v - u0[i])
            outs.append(v)
        for i in range(n):
            grids[i].reshape(5, 12, 12, 12)[:, 2:10, 2:10, 2:10] = outs[i].reshape(5, 8, 8, 8)
    return grids


@pytest.mark.parametrize("exact", [False, True])
def test_gravity_hydro_step_bitwise_vs_oracle(exact):
    f = amr.build_scenario(amr.Scenario.rotating_star, 1, 3)
    st = f.scenario_state(amr.Scenario.rotating_star)
    f.alloc()
    f.set_interior(st)
    lv = forest_leaf_array(f)
    o = O.Oracle()
    t = o.tree([int(p) for p in f.leaves()])
    grids = [np.ascontiguousarray(g) for g in interior_to_ghosted(st)]
    drv = GravityHydroDriver(f, am=True, exact_ghosts=exact)
    dt = 2e-3
    for step in range(2):
        drv.step(dt=dt)
        grids = oracle_gravity_step(o, t, grids, lv, dt)
        got = f.get_interior()
        want = np.stack([g.reshape(5, 12, 12, 12)[:, 2:10, 2:10, 2:10].reshape(5, 512) for g in grids])
        assert got.tobytes() == want.tobytes(), f"step {step}"
    # gravity changes the step: the same step without it differs
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
