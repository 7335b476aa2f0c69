"""AMR regrid with the data on the device vs the
unmodified reference Tree (oracle/_ref/libtmref.so): refine (with cascaded 2:1
refinement) and coarsen carry the grids exactly as Tree::refine / coarsen do
(prolong_cell / restrict_cells, octree.cpp:149-293) — whole ghosted blocks
bitwise; flag_refinement (octree.cpp:295-323) per leaf identical; the host
coarsen topology equals the reference's (CPU)."""
import numpy as np
import pytest

from paper_2412_15518_b200 import amr

from helpers import replay_on_reference


def _tree_pair(ref, lo=1, hi=3):
    f = amr.build_scenario(amr.Scenario.rotating_star, lo, hi)
    t = replay_on_reference(ref, f, 6)
    assert [int(p) for p in t.leaves()] == [int(p) for p in f.leaves()]
    return f, t


def _coarsenable(f):
    """Parents whose 8 children are all leaves, in leaf order."""
    lv = [int(p) for p in f.leaves()]
    have = set(lv)
    out = []
    for p in lv:
        l, i, j, k = amr.unpack(p)
        if l == 0:
            continue
        par = amr.pack(l - 1, i >> 1, j >> 1, k >> 1)
        kids = [amr.pack(l, 2 * (i >> 1) + (b & 1), 2 * (j >> 1) + ((b >> 1) & 1),
                         2 * (k >> 1) + (b >> 2)) for b in range(8)]
        if all(c in have for c in kids) and par not in out:
            out.append(par)
    return out


@pytest.mark.ref
def test_coarsen_topology_equals_reference(ref):
    f, t = _tree_pair(ref)
    done = 0
    for par in _coarsenable(f):
        try:
            t.coarsen(par)
            ok = True
        except RuntimeError:
            ok = False
        if ok:
            f.coarsen(par)
            done += 1
        else:
            with pytest.raises(amr.AmrError):
                f.coarsen(par)
        assert [int(p) for p in t.leaves()] == [int(p) for p in f.leaves()]
    assert done > 0


@pytest.mark.gpu
@pytest.mark.ref
@pytest.mark.parametrize("seed", [0, 1])
def test_regrid_data_bitwise_vs_reference(ref, seed):
    f, t = _tree_pair(ref)
    rng = np.random.default_rng(seed)
    f.alloc()
    grids = rng.uniform(0.5, 2.0, (f.leaf_count(), 5 * 1728))
    f.set_grids(grids)
    for i, p in enumerate(f.leaves()):
        t.grid(int(p))[:] = grids[i]
    lv = [int(p) for p in f.leaves()]
    # refine a few leaves of the coarse levels (their neighbours cascade), then
    # coarsen parents whose 8 children are leaves after the refinements
    refine = [p for p in lv if amr.unpack(p)[0] <= 2][::5][:6]
    for p in refine:
        t.refine(p)
    have = set(int(x) for x in t.leaves())
    coarsen = []
    for p in sorted(have):
        l, i, j, k = amr.unpack(p)
        if l < 2:
            continue
        par = amr.pack(l - 1, i >> 1, j >> 1, k >> 1)
        kids = [amr.pack(l, 2 * (i >> 1) + (b & 1), 2 * (j >> 1) + ((b >> 1) & 1),
                         2 * (k >> 1) + (b >> 2)) for b in range(8)]
        if par not in coarsen and par not in refine and all(c in have for c in kids):
            coarsen.append(par)
    applied = []
    for par in coarsen[:4]:
        try:
            t.coarsen(par)
            applied.append(par)
        except RuntimeError:  # would violate 2:1 balance
            pass
    f.regrid(refine, applied)
    assert [int(p) for p in t.leaves()] == [int(p) for p in f.leaves()]
    got = f.get_grids()
    for i, p in enumerate(f.leaves()):
        assert got[i].tobytes() == t.grid(int(p)).tobytes(), f"leaf {i}"
    assert len(applied) > 0


@pytest.mark.gpu
@pytest.mark.ref
@pytest.mark.parametrize("theta", [0.01, 0.05, 0.2])
def test_flag_refinement_equals_reference(ref, theta):
    f, t = _tree_pair(ref)
    f.alloc()
    st = f.scenario_state(amr.Scenario.rotating_star)
    f.set_interior(st)
    f.fill_ghosts()
    grids = f.get_grids()
    for i, p in enumerate(f.leaves()):
        t.grid(int(p))[:] = grids[i]
    got = f.flag_refinement(theta)
    want = np.array([t.flag(int(p), theta) for p in f.leaves()])
    assert (got == want).all()
    assert 0 < got.sum() < len(got) or theta == 0.2


@pytest.mark.gpu
def test_gravity_hydro_driver_steps_across_a_regrid():
    """Refine during a run: the driver carries the state along (regrid), rebuilds
    the gravity plan, and the next step equals a fresh driver on the regridded
    forest started from the same (regridded) state."""
    from paper_2412_15518_b200.driver import GravityHydroDriver

    def run(regrid_first):
        f = amr.build_scenario(amr.Scenario.rotating_star, 1, 3)
        f.alloc()
        f.set_interior(f.scenario_state(amr.Scenario.rotating_star))
        d = GravityHydroDriver(f)
        d.step(dt=1e-3)
        lv = [int(p) for p in f.leaves()]
        d.regrid(refine=[p for p in lv if amr.unpack(p)[0] == 1][:2])
        state = f.get_grids()
        if regrid_first:
            d.step(dt=1e-3)
            out = f.get_interior()
        else:
            d.close()
            d2 = GravityHydroDriver(f)
            f.set_grids(state)
            d2.step(dt=1e-3)
            out = f.get_interior()
            d2.close()
        return out, f.leaf_count()

    a, na = run(True)
    b, nb = run(False)
    assert na == nb and a.tobytes() == b.tobytes()
