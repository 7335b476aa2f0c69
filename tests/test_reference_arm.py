"""The CPU arm of bench.py (oracle/ref_capi.cpp tmref_gravity_hydro_step):
the reference's own hydro step with self-gravity from the patch-sparse FMM
(oracle/gravity_amr_sparse.c), the workload built on the reference Tree. It is
timed, not the parity target, but it must compute the same step: without floor
hits it equals the oracle composition the GPU is tested against, bit for bit."""
import numpy as np
import pytest

from oracle import oracle as O

from helpers import oracle_gravity_step

pytestmark = pytest.mark.ref


def _tree(ref, lo=1, hi=3):
    t = ref.tree(max_level=hi)
    t.scenario(0, lo, hi, 0.1)
    return t


def test_pure_hydro_equals_reference_hydro_step(ref):
    a, b = _tree(ref), _tree(ref)
    dt, secs = a.gravity_hydro_step(cfl=0.4, workers=4)
    h = ref.encode_header(1, 1.0, 0.0)
    want = 0.4 * min(b.cell_size(int(p) >> 60) / ref.max_wavespeed(h, b.grid(int(p)).copy())
                     for p in b.leaves())
    assert dt == want  # the CFL dt is computed inside the timed call
    b.hydro_step(dt, workers=4)
    for p in a.leaves():
        assert a.grid(int(p)).tobytes() == b.grid(int(p)).tobytes()


@pytest.mark.parametrize("cadence", [1, 3, 6])
def test_gravity_hydro_step_equals_oracle_composition(ref, cadence):
    t = _tree(ref)
    o = O.Oracle()
    lv = t.leaf_levels()
    plan = o.grav_plan(lv)
    grids = [t.grid(int(p)).copy() for p in t.leaves()]
    ot = o.tree([int(p) for p in t.leaves()])
    dt = 2e-3
    t.gravity_hydro_step(dt=dt, cfl=0.0, workers=4, solves_per_step=cadence, plan=plan)
    grids = oracle_gravity_step(o, ot, grids, lv, dt, cadence)
    for g, p in zip(grids, t.leaves()):
        want = g.reshape(5, 12, 12, 12)[:, 2:10, 2:10, 2:10]
        got = t.grid(int(p)).reshape(5, 12, 12, 12)[:, 2:10, 2:10, 2:10]
        assert got.tobytes() == want.tobytes()
