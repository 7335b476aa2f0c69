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
        if t.is_leaf(p):  # not already refined by a 2:1 cascade
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


RK3_W = {1: 1.0, 2: 0.25, 3: 2.0 / 3.0}


def oracle_gravity_step(o, t, grids, lv, dt, cadence=3, gamma=1.4):
    """One gravity + hydro SSP-RK3 step composed from the oracle (test
    infrastructure): AMR FMM specification (gravity_amr_oracle.c, with the
    angular-momentum correction) -> per RK stage: ghost fill
    (tmo_fill_ghosts_sync) -> stage with the gravity source
    (tmo_stage_subgrid_grav) -> rk3_combine (rk3.hpp:18-27). cadence = FMM
    solves per step: 1 on the step's initial state held over the stages; 3 on
    every stage's input; 6 additionally on every stage's provisional density,
    the source moved to the trapezoid (csrc/grav_source.cu, same association).
    grids: list of ghosted [V*S^3] leaf arrays, modified in place."""
    import ctypes as C

    dp = C.POINTER(C.c_double)
    n = len(grids)
    h = 1.0 / (8.0 * 2.0 ** lv[:, 0].astype(np.float64))
    h3 = (h * h * h)[:, None]

    def interior(g):
        return g.reshape(5, 12, 12, 12)[:, 2:10, 2:10, 2:10].reshape(5, 512)

    plan = o.grav_plan(lv)  # the patch-sparse restatement: bitwise the dense one

    def solve(rho):
        _, gf, _ = plan.solve(np.stack(rho) * h3, flags=1)
        return gf

    u0 = [interior(g).copy() for g in grids]
    ga = solve([u[0] for u in u0]) if cadence else None
    bad = (C.c_int * 3)()
    for stage in (1, 2, 3):
        t.fill_ghosts(grids)
        if cadence >= 3 and stage > 1:
            ga = solve([interior(g)[0].copy() for g in grids])
        outs, rts = [], []
        for i in range(n):
            hdr = np.array([1.0, h[i], dt, gamma, 0.0, 0.0, 0.0, 0.0])
            out = np.zeros(5 * 512 + 6 * 5 * 64 + 1)
            gi = np.ascontiguousarray(ga[:, i * 512:(i + 1) * 512]) if cadence else None
            fn = o.lib.tmo_stage_subgrid_grav if cadence else o.lib.tmo_stage_subgrid
            args = [hdr.ctypes.data_as(dp), 8, 2, 5, grids[i].ctypes.data_as(dp)]
            if cadence:
                args.append(gi.ctypes.data_as(dp))
            rc = fn(*args, out.ctypes.data_as(dp), bad)
            assert rc == 0
            v = out[:2560].reshape(5, 512).copy()
            rts.append(v[0].copy())
            if stage == 2:
                v = u0[i] + 0.25 * (v - u0[i])
            elif stage == 3:
                v = u0[i] + (2.0 / 3.0) * (v - u0[i])
            outs.append(v)
        if cadence == 6:
            gb = solve(rts)
            w, hdt = RK3_W[stage], 0.5 * dt
            for i in range(n):
                u = interior(grids[i])
                r = u[0]
                rho = np.where(r < 1e-10, 1e-10, r)
                iu, iv, iw = u[1] / rho, u[2] / rho, u[3] / rho
                sl = slice(i * 512, (i + 1) * 512)
                dgx, dgy, dgz = gb[0, sl] - ga[0, sl], gb[1, sl] - ga[1, sl], gb[2, sl] - ga[2, sl]
                v = outs[i]
                v[1] = v[1] + w * (hdt * (rho * dgx))
                v[2] = v[2] + w * (hdt * (rho * dgy))
                v[3] = v[3] + w * (hdt * (rho * dgz))
                v[4] = v[4] + w * (hdt * (rho * ((iu * dgx + iv * dgy) + iw * dgz)))
        for i in range(n):
            grids[i].reshape(5, 12, 12, 12)[:, 2:10, 2:10, 2:10] = outs[i].reshape(5, 8, 8, 8)
    return grids
