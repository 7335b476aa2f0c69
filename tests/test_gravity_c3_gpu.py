"""Gravity pinned at the bench configuration (BASELINE.json configs[2]) and on
deep forests: the GPU AMR FMM (csrc/gravity_amr.cu) and the gravity + hydro
step against the oracle (our specification, oracle/gravity_amr_oracle.c, and
the composition of tests/helpers.py) at full size, bitwise.

C3 = rotating star, leaf levels 2..5, 5,888 leaves (3.0e6 cells, 6,729
patches, ~6e6 W/X entries) — exactly the state bench.py times."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2412_15518_b200 import amr
from paper_2412_15518_b200 import gravity as G
from paper_2412_15518_b200.driver import GravityHydroDriver

from helpers import interior_to_ghosted, oracle_gravity_step

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c3():
    f = amr.build_scenario(amr.Scenario.rotating_star, 2, 5, 0.1)
    st = f.scenario_state(amr.Scenario.rotating_star)
    assert f.leaf_count() == 5888
    return f, st


def masses_of(lv, rho):
    h = 1.0 / (8.0 * 2.0 ** lv[:, 0].astype(np.float64))
    return rho * (h * h * h)[:, None]


@pytest.mark.parametrize("am", [False, True])
def test_c3_gravity_solve_bitwise(c3, am):
    f, st = c3
    lv = G.forest_leaf_array(f)
    m = masses_of(lv, st[:, 0])
    pr, gr, cnt = O.Oracle().grav_amr(lv, m, flags=1 if am else 0)
    s = G.GravityAMR(lv)
    assert (s.info()[2], s.info()[3]) == cnt
    assert cnt[0] > 5_000_000  # the W/X lists the bench's M2L evaluates
    phi, g = s.solve(m, am=am)
    assert phi.tobytes() == pr.tobytes()
    assert g.tobytes() == gr.tobytes()


@pytest.mark.parametrize("cadence", [3, 1])
def test_c3_gravity_hydro_step_bitwise(c3, cadence):
    """One bench step (CFL dt on the device) at full C3 size vs the oracle
    composition with that dt."""
    f0, st = c3
    f = amr.build_scenario(amr.Scenario.rotating_star, 2, 5, 0.1)
    f.alloc()
    f.set_interior(st)
    lv = G.forest_leaf_array(f)
    drv = GravityHydroDriver(f, am=True, solves_per_step=cadence)
    dt = drv.step()
    o = O.Oracle()
    t = o.tree([int(p) for p in f.leaves()])
    grids = [np.ascontiguousarray(g) for g in interior_to_ghosted(st)]
    grids = oracle_gravity_step(o, t, grids, lv, dt, cadence)
    want = np.stack([g.reshape(5, 12, 12, 12)[:, 2:10, 2:10, 2:10].reshape(5, 512) for g in grids])
    got = f.get_interior()
    assert got.tobytes() == want.tobytes()
    drv.close()


def dwd_deep_forest(max_level=7, radius=0.02):
    """The double-white-dwarf geometry (configs[4]) sub-sampled: uniform level
    2, then every leaf within `radius` of either star centre refined to
    `max_level` (the forest's 2:1 cascade fills the levels between)."""
    f = amr.Forest(max_level=max_level)
    centres = np.array([[0.35, 0.5, 0.5], [0.65, 0.5, 0.5]])
    for level in range(max_level):
        for p in [int(q) for q in f.leaves()]:
            lvl, i, j, k = amr.unpack(p)
            if lvl != level:
                continue
            s = 1.0 / (1 << lvl)
            lo, hi = np.array([i, j, k]) * s, np.array([i + 1, j + 1, k + 1]) * s
            near = np.clip(centres, lo, hi)
            if level < 2 or (np.linalg.norm(near - centres, axis=1) < radius).any():
                if p in set(int(q) for q in f.leaves()):
                    f.refine(p)
    return f


def test_deep_dwd_forest_gravity_bitwise():
    f = dwd_deep_forest()
    lv = G.forest_leaf_array(f)
    assert lv[:, 0].max() == 7 and lv[:, 0].min() == 2
    rng = np.random.default_rng(24)
    rho = rng.uniform(0.1, 1.0, (lv.shape[0], 512))
    m = masses_of(lv, rho)
    pr, gr, cnt = O.Oracle().grav_amr(lv, m, flags=1, sparse=True)
    phi, g = G.GravityAMR(lv).solve(m, am=True)
    assert phi.tobytes() == pr.tobytes()
    assert g.tobytes() == gr.tobytes()


@pytest.mark.parametrize("seed", [3, 8])
def test_deep_unbalanced_forest_gravity_bitwise(seed):
    """Random unbalanced forests to level 6: W/X pairs across jumps of
    several levels (a balanced forest only has jumps of one)."""
    lv = O.random_forest_leaves(np.random.default_rng(seed), base=2, max_level=6, frac=0.12)
    assert lv[:, 0].max() >= 5
    rng = np.random.default_rng(seed)
    m = masses_of(lv, rng.uniform(0.1, 1.0, (lv.shape[0], 512)))
    pr, gr, cnt = O.Oracle().grav_amr(lv, m, flags=1, sparse=True)
    phi, g = G.GravityAMR(lv).solve(m, am=True)
    assert phi.tobytes() == pr.tobytes()
    assert g.tobytes() == gr.tobytes()
