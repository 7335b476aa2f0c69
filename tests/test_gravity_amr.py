"""AMR FMM gravity specification (oracle/gravity_amr_oracle.c, parity unpinned:
the reference has no gravity code) pinned on CPU against the uniform
specification (bitwise), direct O(N^2) summation, and the conservation laws
(PAPER.md:233)."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O

dp = C.POINTER(C.c_double)


def star_rho(x):
    r2 = ((x - 0.5) ** 2).sum(1)
    return np.maximum(1 - r2 / 0.3 ** 2, 0) ** 1.5 + 1e-3


def masses(leaves, kind="star", seed=0):
    x = O.leaf_centres(leaves)
    h = 1.0 / (8.0 * 2.0 ** leaves[:, 0].astype(np.float64))
    vol = np.repeat(h ** 3, 512)
    if kind == "star":
        rho = star_rho(x)
    else:
        rho = np.random.default_rng(seed).uniform(0.1, 1.0, x.shape[0])
    return (rho * vol).reshape(-1, 512)


def uniform_leaves(level):
    n = 1 << level
    out = []
    def rec(l, i, j, k):
        if l == level:
            out.append((l, i, j, k))
            return
        for c in range(8):
            rec(l + 1, 2 * i + (c & 1), 2 * j + ((c >> 1) & 1), 2 * k + (c >> 2))
    rec(0, 0, 0, 0)
    assert len(out) == n ** 3
    return np.array(out, dtype=np.int32)


def test_uniform_forest_equals_uniform_spec_bitwise():
    o = O.Oracle()
    L = o.lib
    L.tmo_grav_solve.argtypes = [C.c_int, dp, dp, dp]
    lv = uniform_leaves(1)  # cell depth 4, 16^3 cells
    m = masses(lv, "random", 3)
    phi, g, cnt = o.grav_amr(lv, m)
    assert cnt == (0, 0)
    # uniform spec works on the global (k,j,i) grid
    N = 16
    gl = (O.leaf_centres(lv) * N - 0.5).round().astype(np.int64)
    gidx = (gl[:, 2] * N + gl[:, 1]) * N + gl[:, 0]
    mu = np.zeros(N ** 3)
    mu[gidx] = m.reshape(-1)
    pu, gu = np.zeros(N ** 3), np.zeros(3 * N ** 3)
    L.tmo_grav_solve(4, mu.ctypes.data_as(dp), pu.ctypes.data_as(dp), gu.ctypes.data_as(dp))
    assert np.array_equal(phi, pu[gidx])
    assert np.array_equal(g, gu.reshape(3, -1)[:, gidx])


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_amr_fmm_vs_direct_and_momentum(seed):
    o = O.Oracle()
    rng = np.random.default_rng(seed)
    lv = O.random_forest_leaves(rng, base=1, max_level=3, frac=0.25)
    assert len(set(lv[:, 0])) > 1
    m = masses(lv, "star" if seed % 2 == 0 else "random", seed)
    phi, g, cnt = o.grav_amr(lv, m)
    assert cnt[0] > 0 and cnt[1] > 0
    pd, gd, _ = o.grav_amr(lv, m, direct=True)
    # order-2 expansions; unbalanced trees put W/X pairs at 1.5 cell widths
    assert np.max(np.abs(phi - pd) / np.abs(pd)) < 3e-2
    gm = np.sqrt((gd ** 2).sum(0))
    err = np.sqrt(((g - gd) ** 2).sum(0))
    # uniform level-2 star: 2.1e-2 / 3.8e-2 — the AMR tree is no worse
    assert np.sqrt(np.mean(err ** 2)) / np.sqrt(np.mean(gm ** 2)) < 5e-2
    F = g * m.reshape(-1)  # every interaction pair is mutual and exactly opposite
    assert np.abs(F.sum(1)).max() <= 1e-13 * np.abs(F).sum(1).max()


@pytest.mark.parametrize("seed", [0, 3])
def test_every_leaf_cell_pair_interacts_exactly_once(seed):
    """Count mode (flags & 2): each M2L adds the source's cell count, each P2P
    adds 1; every leaf cell must see exactly n - 1 others."""
    o = O.Oracle()
    lv = O.random_forest_leaves(np.random.default_rng(seed), base=1, max_level=3, frac=0.25)
    n = lv.shape[0] * 512
    phi, _, cnt = o.grav_amr(lv, np.ones((lv.shape[0], 512)), flags=2)
    assert cnt[0] > 0 and cnt[1] > 0
    assert np.all(phi == n - 1)


def torque(g, m, x, about):
    r = x - about
    return (np.cross(r, (g * m).T)).sum(0)


def test_angular_momentum_correction():
    o = O.Oracle()
    rng = np.random.default_rng(7)
    lv = O.random_forest_leaves(rng, base=1, max_level=3, frac=0.25)
    m = masses(lv, "random", 7)
    x = O.leaf_centres(lv)
    mm = m.reshape(-1)
    com = (x * mm[:, None]).sum(0) / mm.sum()
    _, g0, _ = o.grav_amr(lv, m, flags=0)
    _, g1, _ = o.grav_amr(lv, m, flags=1)
    scale = (np.linalg.norm(x - com, axis=1) * np.linalg.norm(g0, axis=0) * mm).sum()
    t0 = np.abs(torque(g0, mm, x, com)).max() / scale
    t1 = np.abs(torque(g1, mm, x, com)).max() / scale
    assert t0 > 1e-8  # truncated M2L forces are not central
    assert t1 < 1e-14  # corrected to round-off
    F1 = (g1 * mm).sum(1)
    assert np.abs(F1).max() <= 1e-13 * np.abs(g1 * mm).sum(1).max()
    assert np.max(np.abs(g1 - g0)) < 1e-2 * np.max(np.abs(g0))


def test_am_correct_restated_in_numpy():
    """tmo_grav_am_correct's rigid-rotation field, recomputed with numpy."""
    o = O.Oracle()
    rng = np.random.default_rng(9)
    lv = O.random_forest_leaves(rng, base=1, max_level=2, frac=0.3)
    m = masses(lv, "random", 9).reshape(-1)
    x = O.leaf_centres(lv)
    g = rng.normal(size=(3, m.size))
    g2 = g.copy()
    S = np.zeros(16)
    w = np.zeros(3)
    o.lib.tmo_grav_am_correct(lv.shape[0], m.ctypes.data_as(dp), np.ascontiguousarray(x).ctypes.data_as(dp),
                              g2.ctypes.data_as(dp), S.ctypes.data_as(dp), w.ctypes.data_as(dp))
    com = (x * m[:, None]).sum(0) / m.sum()
    r = x - com
    tau = np.cross(r, (g * m).T).sum(0)
    J = (m[:, None, None] * ((r * r).sum(1)[:, None, None] * np.eye(3) - r[:, :, None] * r[:, None, :])).sum(0)
    w_np = np.linalg.solve(J, -tau)
    assert np.allclose(w, w_np, rtol=1e-10, atol=1e-14 * np.abs(w_np).max())
    assert np.allclose(g2, g + np.cross(w_np, r).T, rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("seed", [0, 1, 4])
def test_product_plan_pairs_match_spec(seed):
    """The product's host plan (csrc/gravity_amr_plan.cpp) generates exactly
    the specification's W/X and cross-depth U pair counts."""
    from paper_2412_15518_b200 import gravity as G

    o = O.Oracle()
    lv = O.random_forest_leaves(np.random.default_rng(seed), base=1, max_level=3, frac=0.3)
    _, _, cnt = o.grav_amr(lv, np.ones((lv.shape[0], 512)), flags=2)
    info = G.amr_plan_info(lv)
    assert (info[2], info[3]) == cnt
    assert info[0] == lv[:, 0].max() + 1


def test_product_plan_rejects_bad_leaves():
    from paper_2412_15518_b200 import gravity as G
    lv = uniform_leaves(1)
    with pytest.raises(ValueError, match="tile"):
        G.amr_plan_info(lv[:-1])
    with pytest.raises(ValueError, match="overlap"):
        G.amr_plan_info(np.concatenate([lv, [[0, 0, 0, 0]]]))


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_let_plan_pairwise_consistent(world):
    """Multipole-moment exchange (LET, csrc grav_let_plan): rank r's send list to
    q is q's receive list from r (counts and ordered hashes), and the owned
    internal patches of all ranks plus the shared top cover every internal patch."""
    from paper_2412_15518_b200 import amr, dist
    from paper_2412_15518_b200.gravity import amr_let_plan, amr_plan_info, forest_leaf_array

    f = amr.build_scenario(amr.Scenario.rotating_star, 2, 4)
    lv = forest_leaf_array(f)
    owner = np.array(dist.partition(f, world))
    b = np.searchsorted(owner, np.arange(world + 1))
    b[-1] = len(owner)
    plans = [amr_let_plan(lv, b, r) for r in range(world)]
    for r in range(world):
        assert plans[r]["send"][r] == 0 and plans[r]["recv"][r] == 0
        for q in range(world):
            assert plans[r]["send"][q] == plans[q]["recv"][r]
            assert plans[r]["send_hash"][q] == plans[q]["recv_hash"][r]
    tops = {p["top_internal"] for p in plans}
    assert len(tops) == 1  # every rank computes the same shared top
    nodes = amr_plan_info(lv)[1]
    leaves = lv.shape[0]
    assert sum(p["owned_internal"] for p in plans) + tops.pop() == nodes - leaves


# ---- the patch-sparse restatement (oracle/gravity_amr_sparse.c): the same
# specification with per-patch storage, tabulated geometry, SIMD V lists and
# per-target list buckets — the CPU baseline and the oracle for deep forests

def _fast_builds():
    out = [False]
    if O.host_has_avx2_fma():
        out.append(True)
    return out


@pytest.mark.parametrize("fast", _fast_builds())
@pytest.mark.parametrize("seed", [0, 1, 4, 9])
@pytest.mark.parametrize("flags", [0, 1, 2])
def test_sparse_restatement_bitwise_equals_dense(fast, seed, flags):
    dense = O.Oracle(fast=False)
    o = O.Oracle(fast=fast)
    lv = O.random_forest_leaves(np.random.default_rng(seed), base=1, max_level=4, frac=0.3)
    m = masses(lv, "star" if seed % 2 else "random", seed)
    a = dense.grav_amr(lv, m, flags=flags)
    b = o.grav_amr(lv, m, flags=flags, sparse=True)
    assert a[2] == b[2]
    assert a[0].tobytes() == b[0].tobytes() and a[1].tobytes() == b[1].tobytes()


def test_sparse_plan_reused_across_solves():
    o = O.Oracle()
    lv = O.random_forest_leaves(np.random.default_rng(5), base=2, max_level=4, frac=0.2)
    plan = o.grav_plan(lv)
    for seed in (1, 2):
        m = masses(lv, "random", seed)
        a = o.grav_amr(lv, m, flags=1)
        b = plan.solve(m, flags=1)
        assert a[0].tobytes() == b[0].tobytes() and a[1].tobytes() == b[1].tobytes()


def test_sparse_deep_forest_count_mode_and_accuracy():
    """Leaf level 7 (cell depth 10), beyond the dense restatement's reach:
    every leaf-cell pair is covered exactly once (count mode), and the field
    agrees with direct summation like the shallow forests do."""
    o = O.Oracle()
    rng = np.random.default_rng(21)
    lv = O.random_forest_leaves(rng, base=1, max_level=7, frac=0.22)
    assert lv[:, 0].max() == 7
    n = lv.shape[0] * 512
    ones = np.ones((lv.shape[0], 512))
    phi, _, _ = o.grav_amr(lv, ones, flags=2, sparse=True)
    assert (phi == n - 1).all()
    if n <= 40_000:
        m = masses(lv, "star")
        p, g, _ = o.grav_amr(lv, m, flags=0, sparse=True)
        pd, gd, _ = o.grav_amr(lv, m, direct=True)
        assert np.abs(p - pd).max() / np.abs(pd).max() < 3e-2


def test_sparse_rejects_bad_tilings():
    o = O.Oracle()
    lv = np.array([[1, 0, 0, 0], [1, 1, 0, 0]], dtype=np.int32)  # 2 of 8 octants
    with pytest.raises(ValueError):
        o.grav_amr(lv, np.ones((2, 512)), sparse=True)
    lv = np.array([[0, 0, 0, 0], [1, 0, 0, 0]], dtype=np.int32)  # overlap
    with pytest.raises(ValueError):
        o.grav_amr(lv, np.ones((2, 512)), sparse=True)
