"""AMR FMM gravity on the GPU (csrc/gravity_amr.cu) vs our specification
(oracle/gravity_amr_oracle.c): bitwise, with and without the angular-momentum
correction, from host masses and from a forest's device arena."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2412_15518_b200 import amr
from paper_2412_15518_b200 import gravity as G

from test_gravity_amr import masses, uniform_leaves

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [0, 1, 2, 5])
@pytest.mark.parametrize("am", [False, True])
def test_amr_gravity_bitwise_vs_spec(seed, am):
    o = O.Oracle()
    lv = O.random_forest_leaves(np.random.default_rng(seed), base=1, max_level=3, frac=0.25)
    m = masses(lv, "star" if seed % 2 == 0 else "random", seed)
    pr, gr, cnt = o.grav_amr(lv, m, flags=1 if am else 0)
    s = G.GravityAMR(lv)
    info = s.info()
    assert (info[2], info[3]) == cnt
    phi, g = s.solve(m, am=am)
    assert phi.tobytes() == pr.tobytes()
    assert g.tobytes() == gr.tobytes()


def test_amr_gravity_uniform_forest_equals_uniform_solver():
    lv = uniform_leaves(2)  # 32^3 cells
    m = masses(lv, "random", 4)
    phi, g = G.GravityAMR(lv).solve(m)
    N = 32
    gl = (O.leaf_centres(lv) * N - 0.5).round().astype(np.int64)
    gidx = (gl[:, 2] * N + gl[:, 1]) * N + gl[:, 0]
    mu = np.zeros(N ** 3)
    mu[gidx] = m.reshape(-1)
    pu, gu = G.GravitySolver(5).solve(mu)
    assert phi.tobytes() == pu[gidx].tobytes()
    assert g.tobytes() == gu[:, gidx].tobytes()


def test_amr_gravity_from_forest_arena_device_path():
    import torch

    f = amr.build_scenario(amr.Scenario.rotating_star, 1, 3)
    f.alloc()
    st = f.scenario_state(amr.Scenario.rotating_star)
    f.set_interior(st)
    lv = G.forest_leaf_array(f)
    h = 1.0 / (8.0 * 2.0 ** lv[:, 0].astype(np.float64))
    m = st[:, 0, :] * (h * h * h)[:, None]
    o = O.Oracle()
    pr, gr, _ = o.grav_amr(lv, m, flags=1)
    s = G.GravityAMR(lv)
    s.mass_from_arena(f)
    phi, g = s.solve(None, am=True, phi=torch.empty(lv.shape[0] * 512, dtype=torch.float64, device="cuda"))
    torch.cuda.synchronize()
    assert phi.cpu().numpy().tobytes() == pr.tobytes()
    assert g.cpu().numpy().tobytes() == gr.tobytes()
    stats = s.am_stats()
    x = O.leaf_centres(lv)
    mm = m.reshape(-1)
    gg = g.cpu().numpy()
    tq = np.cross(x - stats[:3], (gg * mm).T).sum(0)
    scale = (np.linalg.norm(x - stats[:3], axis=1) * np.linalg.norm(gg, axis=0) * mm).sum()
    assert np.abs(tq).max() / scale < 1e-14


@pytest.mark.parametrize("am", [False, True])
def test_amr_gravity_single_leaf_root(am):
    """Edge case: the whole domain one leaf (level 0): the root patch is a leaf,
    its locals come from the dense levels' L2L and its own V sums."""
    o = O.Oracle()
    lv = np.array([[0, 0, 0, 0]], dtype=np.int32)
    m = masses(lv, "random", 11)
    pr, gr, cnt = o.grav_amr(lv, m, flags=1 if am else 0)
    phi, g = G.GravityAMR(lv).solve(m, am=am)
    assert phi.tobytes() == pr.tobytes()
    assert g.tobytes() == gr.tobytes()


def test_amr_gravity_level1_uniform():
    """Edge case: eight level-1 leaves (every patch a leaf, one internal root)."""
    o = O.Oracle()
    lv = uniform_leaves(1)
    m = masses(lv, "star", 12)
    pr, gr, _ = o.grav_amr(lv, m, flags=1)
    phi, g = G.GravityAMR(lv).solve(m, am=True)
    assert phi.tobytes() == pr.tobytes()
    assert g.tobytes() == gr.tobytes()
