"""Bit-exact indexing: our host forest vs the UNMODIFIED reference Tree (CPU).

Morton keys, NodeId packing, canonical leaf order, face-neighbour resolution
(incl. periodic wrap, reflective walls, finer-quadrant order), ghost-fill
plans, 2:1 balance and partition_leaves must be identical.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2412_15518_b200 import amr

from helpers import replay_on_reference


def test_morton_kats():
    """test_amr.cpp:75-96."""
    assert amr.morton_encode(1, 1, 0, 1) == 5
    assert amr.morton_encode(0, 0, 0, 0) == 0
    with pytest.raises(amr.AmrError):
        amr.morton_encode(1, 2, 0, 0)
    with pytest.raises(amr.AmrError):
        amr.morton_encode(3, 0, 8, 0)
    rng = np.random.default_rng(5)
    for _ in range(500):
        level = int(rng.integers(1, 11))
        m = (1 << level) - 1
        i, j, k = (int(x) & m for x in rng.integers(0, 2 ** 30, 3))
        key = amr.morton_encode(level, i, j, k)
        assert amr.morton_decode(level, key) == (i, j, k)


def test_partition_kats():
    """test_amr.cpp:414-455."""
    assert amr.partition_leaves([512] * 8, 2) == [0, 0, 0, 0, 1, 1, 1, 1]
    assert amr.partition_leaves([7, 1, 1, 1], 2) == [0, 1, 1, 1]
    with pytest.raises(amr.AmrError):
        amr.partition_leaves([1, 1], 3)
    rng = np.random.default_rng(7)
    for _ in range(200):
        n = 1 + int(rng.integers(0, 64))
        L = 1 + int(rng.integers(0, min(n, 8)))
        w = [1 + int(x) for x in rng.integers(0, 1000, n)]
        owner = amr.partition_leaves(w, L)
        load = [0] * L
        for i, o in enumerate(owner):
            assert 0 <= o < L and (i == 0 or o >= owner[i - 1])
            load[o] += w[i]
        for r in range(L):
            assert 0 < load[r] <= sum(w) // L + max(w)


@pytest.mark.ref
def test_morton_and_partition_vs_reference(ref):
    rng = np.random.default_rng(11)
    a = np.zeros(1, np.uint64)
    for _ in range(300):
        level = int(rng.integers(0, 21))
        m = (1 << level) - 1
        i, j, k = (int(x) & m for x in rng.integers(0, 2 ** 40, 3))
        ref.lib.tmref_morton_encode(level, i, j, k, O.u64ptr(a))
        assert amr.morton_encode(level, i, j, k) == int(a[0])
        assert amr.morton_dfs_rank(level, int(a[0])) == ref.lib.tmref_morton_dfs_rank(level, int(a[0]))
    import ctypes as C
    for _ in range(300):
        n = int(rng.integers(1, 100))
        L = int(rng.integers(1, min(n, 9) + 1))
        w = rng.integers(1, 2 ** 40, n).astype(np.uint64)
        o = np.zeros(n, np.int32)
        ref.lib.tmref_partition_leaves(O.u64ptr(w), n, L, o.ctypes.data_as(C.POINTER(C.c_int)))
        assert amr.partition_leaves(w, L) == o.tolist()


def _random_pair(ref, rng, max_level, refines, bc, root):
    t = ref.tree(max_level=max_level, bc=bc, root_dims=root)
    f = amr.Forest(max_level=max_level, bc=bc, root_dims=root)
    for _ in range(refines):
        lv = t.leaves()
        cand = [int(p) for p in lv if (int(p) >> 60) < max_level]
        if not cand:
            break
        pick = cand[int(rng.integers(0, len(cand)))]
        t.refine(pick)
        f.refine(pick)
    return t, f


@pytest.mark.ref
@pytest.mark.parametrize("seed,bc,root,refines", [
    (1, (0, 0, 0), (1, 1, 1), 8), (2, (1, 0, 1), (1, 1, 1), 10), (3, (0, 1, 0), (2, 1, 1), 8),
    (4, (1, 1, 1), (1, 2, 3), 12), (5, (0, 0, 0), (1, 1, 1), 30)])
def test_forest_matches_reference_tree(ref, seed, bc, root, refines):
    rng = np.random.default_rng(seed)
    t, f = _random_pair(ref, rng, 4, refines, bc, root)
    assert (f.leaves() == t.leaves()).all()
    assert f.is_balanced() and t.balanced()
    for p in f.leaves():
        for axis in range(3):
            for d in (-1, 1):
                k1, ids1 = f.face_neighbor(int(p), axis, d)
                k2, ids2 = t.face_neighbor(int(p), axis, d)
                assert int(k1) == k2 and ids1 == ids2
    for axis in range(3):
        assert (f.plan(axis) == t.plan(axis)).all()
    for lvl in range(5):
        assert f.cell_size(lvl) == t.cell_size(lvl)


@pytest.mark.ref
@pytest.mark.parametrize("kind,lo,hi,bc", [(amr.Scenario.rotating_star, 2, 4, (0, 0, 0)),
                                           (amr.Scenario.sod, 2, 4, (0, 1, 1)),
                                           (amr.Scenario.sedov, 2, 4, (0, 0, 0))])
def test_scenario_topology_vs_reference(ref, kind, lo, hi, bc):
    f = amr.build_scenario(kind, lo, hi, bc=bc)
    assert f.is_balanced()
    t = replay_on_reference(ref, f, hi, bc)
    assert (f.leaves() == t.leaves()).all()


def test_named_config_sizes():
    """Leaf counts of the BASELINE configs (uniform L2 / L4, 5-level star)."""
    f2 = amr.build_scenario(amr.Scenario.rotating_star, 2, 2)
    assert f2.leaf_count() == 64
    f4 = amr.build_scenario(amr.Scenario.rotating_star, 4, 4)
    assert f4.leaf_count() == 4096
    f5 = amr.build_scenario(amr.Scenario.rotating_star, 2, 5)
    assert f5.is_balanced()
    levels = np.array([amr.unpack(int(p))[0] for p in f5.leaves()])
    # 5,888 leaves (L2:8, L3:288, L4:664, L5:4,928)
    assert f5.leaf_count() == 5888
    assert np.bincount(levels, minlength=6)[2:].tolist() == [8, 288, 664, 4928]
    assert amr.build_scenario(amr.Scenario.sod, 2, 6, bc=(0, 1, 1)).leaf_count() == 19104
    assert amr.build_scenario(amr.Scenario.sedov, 2, 6).leaf_count() == 6672
    assert amr.build_scenario(amr.Scenario.double_white_dwarf, 2, 7).leaf_count() == 228824


def test_scenario_state_is_deterministic():
    f = amr.build_scenario(amr.Scenario.rotating_star, 2, 3)
    a = f.scenario_state(amr.Scenario.rotating_star, 7)
    b = f.scenario_state(amr.Scenario.rotating_star, 7)
    assert a.tobytes() == b.tobytes()
    assert np.all(a[:, 0] > 0) and np.isfinite(a).all()


@pytest.mark.parametrize("kind,lo,hi,bc", [(amr.Scenario.rotating_star, 2, 5, (0, 0, 0)),
                                           (amr.Scenario.double_white_dwarf, 2, 5, (0, 0, 0)),
                                           (amr.Scenario.sod, 2, 5, (0, 1, 1)),
                                           (amr.Scenario.sedov, 2, 5, (0, 0, 0))])
def test_scenarios_built_on_the_reference_tree_match(ref, kind, lo, hi, bc):
    """bench.py's reference arm builds its workload on the reference Tree
    (oracle/ref_capi.cpp tmref_tree_scenario/_fill): the same leaves in the
    same order and the same initial state, bit for bit, as the product's
    scenario (csrc/scenario.cpp) the GPU arm times."""
    t = ref.tree(max_level=hi, bc=bc)
    t.scenario(int(kind), lo, hi, 0.1)
    f = amr.build_scenario(kind, lo, hi, 0.1, bc=bc)
    assert np.array_equal(t.leaves(), np.array(f.leaves(), dtype=np.uint64))
    st = f.scenario_state(kind)
    for i, p in enumerate(f.leaves()):
        g = t.grid(int(p)).reshape(5, 12, 12, 12)
        assert g[:, 2:10, 2:10, 2:10].reshape(5, 512).tobytes() == st[i].tobytes()
        assert not g[:, :2].any()  # ghosts zero
    lv = t.leaf_levels()
    assert [tuple(r) for r in lv[:3]] == [amr.unpack(int(p)) for p in f.leaves()[:3]]
