"""Shared test helpers (test infrastructure)."""
import numpy as np

from paper_2412_15518_b200 import amr


def replay_on_reference(ref, f, max_level, bc=(0, 0, 0), root_dims=(1, 1, 1)):
    """Rebuild a forest topology inside the reference Tree by refining every
    internal node in level order (cascades only touch nodes internal in ours)."""
    internal = set()
    for p in f.leaves():
        lvl, ci, cj, ck = amr.unpack(int(p))
        for l in range(lvl):
            s = lvl - l
            internal.add(amr.pack(l, ci >> s, cj >> s, ck >> s))
    t = ref.tree(max_level=max_level, bc=bc, root_dims=root_dims)
    for p in sorted(internal, key=lambda q: (q >> 60, q)):
        if p in set(int(x) for x in t.leaves()):
            t.refine(p)
    return t


def interior_to_ghosted(compact, edge=8, ghost=2):
    """compact [n][V][E^3] -> ghosted [n][V*S^3] with zero ghosts."""
    n, V, _ = compact.shape
    S = edge + 2 * ghost
    g = np.zeros((n, V, S, S, S))
    g[:, :, ghost:ghost + edge, ghost:ghost + edge, ghost:ghost + edge] = compact.reshape(n, V, edge, edge, edge)
    return g.reshape(n, -1)


def stage_visible_mask(vars_=5, edge=8, ghost=2):
    """Cells the stage reads: interior + face ghosts (at most one coordinate
    outside the interior range), as a flat mask over [V][S][S][S]."""
    S = edge + 2 * ghost
    r = np.arange(S)
    out = (r < ghost) | (r >= ghost + edge)
    nout = out[:, None, None].astype(int) + out[None, :, None] + out[None, None, :]
    return np.broadcast_to(nout <= 1, (vars_, S, S, S)).reshape(-1)


def interior_mask(vars_=5, edge=8, ghost=2):
    """Interior cells of a flat ghosted [V][S][S][S] block."""
    S = edge + 2 * ghost
    r = np.arange(S)
    inn = (r >= ghost) & (r < ghost + edge)
    m = inn[:, None, None] & inn[None, :, None] & inn[None, None, :]
    return np.broadcast_to(m, (vars_, S, S, S)).reshape(-1)
