"""The oracle restatement vs golden outputs of the UNMODIFIED reference
(tests/golden/reference_golden.npz, made by tests/golden/make_golden.py from
oracle/_ref/libtmref.so). Needs only liboracle.so, not the reference sources."""
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def test_stage_golden(orc, gold):
    rc, out, _ = orc.stage_fused(np.ascontiguousarray(gold["euler_in"]), 4)
    assert rc == 0 and out.tobytes() == gold["euler_out"].tobytes()
    rc, out, _ = orc.stage_fused(np.ascontiguousarray(gold["scalar_in"]), 2, vars=1)
    assert rc == 0 and out.tobytes() == gold["scalar_out"].tobytes()


def test_ghost_fill_and_plan_golden(orc, gold):
    leaves = gold["leaves"]
    t = orc.tree(leaves, bc=tuple(int(b) for b in gold["bc"]))
    assert (t.leaves() == leaves).all()
    for a in range(3):
        assert (t.plan(a) == gold[f"plan{a}"]).all()
    S = 12
    grids = []
    for i in range(len(leaves)):
        g = np.zeros((5, S, S, S))
        g[:, 2:10, 2:10, 2:10] = gold["interiors"][i].reshape(5, 8, 8, 8)
        grids.append(np.ascontiguousarray(g.reshape(-1)))
    t.fill_ghosts(grids)
    for g in grids:
        g.reshape(5, S, S, S)[:, 2:10, 2:10, 2:10] *= 1.01
    t.fill_ghosts(grids)
    for i, g in enumerate(grids):
        assert g.tobytes() == gold["grids"][i].tobytes()
