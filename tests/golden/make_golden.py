"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref/libtmref.so,
built in place from /root/reference/proj by oracle/Makefile). Run here, where the
reference exists; the fixtures let the oracle restatement be pinned on machines
without the reference sources.

  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    ref = O.Ref()
    rng = np.random.default_rng(20241218)
    # --- stage: 4 Euler slices (mixed dx) + 2 scalar slices, reference outputs
    S = 12
    ins5, ins1 = 8 + 5 * S ** 3, 8 + S ** 3
    e_in = np.zeros(4 * ins5)
    for s in range(4):
        dx = (1 / 64) * 2.0 ** -s
        e_in[s * ins5:s * ins5 + 8] = ref.encode_header(1, dx, 0.2 * dx)
        e_in[s * ins5 + 8:(s + 1) * ins5] = O.random_state(rng)
    rc, e_out, _ = ref.stage_fused(e_in, 4)
    assert rc == 0
    s_in = np.zeros(2 * ins1)
    for s in range(2):
        s_in[s * ins1:s * ins1 + 8] = ref.encode_header(0, 0.05, 0.002, advect=(0.7, 0.1, -0.3))
        s_in[s * ins1 + 8:(s + 1) * ins1] = rng.uniform(0.2, 2.0, S ** 3)
    rc, s_out, _ = ref.stage_fused(s_in, 2, vars=1)
    assert rc == 0
    # --- ghost fill on a 2-level tree (full ghosted arrays after 2 exchanges)
    t = ref.tree(max_level=3, bc=(0, 1, 0))
    t.refine(O.pack(0, 0, 0, 0))
    t.refine(O.pack(1, 0, 0, 0))
    t.refine(O.pack(1, 1, 1, 1))
    leaves = t.leaves()
    interiors = rng.uniform(0.5, 2.0, (len(leaves), 5, 512))
    for i, p in enumerate(leaves):
        g = t.grid(int(p)).reshape(5, S, S, S)
        g[:] = 0.0
        g[:, 2:10, 2:10, 2:10] = interiors[i].reshape(5, 8, 8, 8)
    t.fill_ghosts()
    for i, p in enumerate(leaves):  # second exchange after a change (history-dependent prolongation)
        g = t.grid(int(p)).reshape(5, S, S, S)
        g[:, 2:10, 2:10, 2:10] *= 1.01
    t.fill_ghosts()
    grids = np.stack([t.grid(int(p)).copy() for p in leaves])
    plans = [t.plan(a) for a in range(3)]
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), euler_in=e_in, euler_out=e_out,
                        scalar_in=s_in, scalar_out=s_out, leaves=leaves, bc=np.array([0, 1, 0]),
                        interiors=interiors, grids=grids, plan0=plans[0], plan1=plans[1],
                        plan2=plans[2])
    print("wrote", os.path.join(HERE, "reference_golden.npz"))


if __name__ == "__main__":
    main()
