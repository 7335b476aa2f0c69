"""FMM gravity on a uniform cell level.

The reference has no gravity code, so the algorithm is our own
specification, restated in oracle/gravity_oracle.c and matched
bitwise by the sm_100a kernels (csrc/gravity.cu): order-2 Cartesian
multipoles, the 189-cell same-level interaction stencil (M2L, Dehnen
truncation -> exact linear-momentum conservation), L2L, and the 26-neighbour
monopole near field (P2P) fused with L2P.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import TmgpuError, lib

_vp = C.c_void_p
_ep = C.POINTER(TmgpuError)
lib.tmgpu_gravity_create.restype = _vp
lib.tmgpu_gravity_create.argtypes = [C.c_int, _ep]
lib.tmgpu_gravity_destroy.restype = None
lib.tmgpu_gravity_destroy.argtypes = [_vp]
lib.tmgpu_gravity_solve.restype = C.c_int
lib.tmgpu_gravity_solve.argtypes = [_vp, _vp, _vp, _vp, C.c_int, _vp, _ep]
lib.tmgpu_gravity_mass_from_arena.restype = C.c_int
lib.tmgpu_gravity_mass_from_arena.argtypes = [_vp, _vp, _vp, C.c_longlong, C.c_int, C.c_double,
                                              _vp, _ep]


class GravitySolver:
    """FMM on a uniform level of N = 2^D cells per axis (unit box)."""

    def __init__(self, D: int):
        err = TmgpuError()
        self.D, self.N = D, 1 << D
        self.h = lib.tmgpu_gravity_create(D, C.byref(err))
        if not self.h:
            _lib.check(err.code or _lib.TMGPU_ERR_CUDA, err)

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:  # lib is None at interpreter exit
            lib.tmgpu_gravity_destroy(self.h)
            self.h = None

    def solve(self, mass):
        """mass: N^3 finest-level masses, (k,j,i) order (numpy: host path;
        CUDA tensor: device path). Returns (phi[N^3], g[3, N^3])."""
        n3 = self.N ** 3
        err = TmgpuError()
        if isinstance(mass, np.ndarray):
            m = np.ascontiguousarray(mass, dtype=np.float64).reshape(-1)
            if m.size != n3:
                raise ValueError("mass must have N^3 entries")
            phi, g = np.zeros(n3), np.zeros(3 * n3)
            _lib.check(lib.tmgpu_gravity_solve(self.h, m.ctypes.data, phi.ctypes.data,
                                               g.ctypes.data, _lib.TMGPU_HOST_PTRS, None,
                                               C.byref(err)), err)
            return phi, g.reshape(3, -1)
        import torch

        phi = torch.empty(n3, dtype=torch.float64, device=mass.device)
        g = torch.empty(3 * n3, dtype=torch.float64, device=mass.device)
        st = torch.cuda.current_stream(mass.device).cuda_stream
        _lib.check(lib.tmgpu_gravity_solve(self.h, mass.data_ptr(), phi.data_ptr(), g.data_ptr(),
                                           0, st, C.byref(err)), err)
        return phi, g.view(3, -1)

    def solve_forest(self, forest, phi, g, stream=None, sync=True):
        """Gravity of a uniform forest's device state (rho -> masses -> FMM)
        into device tensors phi[N^3], g[3*N^3]."""
        import torch

        if getattr(self, "_ijk_for", None) != id(forest):
            from .amr import unpack

            leaves = [unpack(int(p)) for p in forest.local_leaves()]
            if {lv[0] for lv in leaves} != {self.D - 3}:
                raise ValueError("gravity needs a uniform forest at level D - 3")
            ijk = np.array([lv[1:] for lv in leaves], dtype=np.int32).reshape(-1)
            self._ijk = torch.from_numpy(ijk).cuda()
            self._ijk_for = id(forest)
        hc = 1.0 / self.N
        err = TmgpuError()
        _lib.check(lib.tmgpu_gravity_mass_from_arena(self.h, forest.arena_ptr(),
                                                     self._ijk.data_ptr(), forest.local_count(),
                                                     forest.vars, hc * hc * hc, stream,
                                                     C.byref(err)), err)
        _lib.check(lib.tmgpu_gravity_solve(self.h, None, phi.data_ptr(), g.data_ptr(),
                                           0 if sync else _lib.TMGPU_ASYNC, stream, C.byref(err)),
                   err)


_lp = C.POINTER(C.c_longlong)
lib.tmgpu_gravity_amr_create.restype = _vp
lib.tmgpu_gravity_amr_create.argtypes = [_vp, C.c_longlong, _ep]
lib.tmgpu_gravity_amr_destroy.restype = None
lib.tmgpu_gravity_amr_destroy.argtypes = [_vp]
lib.tmgpu_gravity_amr_info.restype = C.c_int
lib.tmgpu_gravity_amr_info.argtypes = [_vp, _lp]
lib.tmgpu_gravity_amr_plan_info.restype = C.c_int
lib.tmgpu_gravity_amr_plan_info.argtypes = [_vp, C.c_longlong, _lp, _ep]
lib.tmgpu_gravity_amr_mass_from_arena.restype = C.c_int
lib.tmgpu_gravity_amr_mass_from_arena.argtypes = [_vp, _vp, C.c_int, _vp, _ep]
lib.tmgpu_gravity_amr_solve.restype = C.c_int
lib.tmgpu_gravity_amr_solve.argtypes = [_vp, _vp, _vp, _vp, C.c_int, _vp, _ep]
lib.tmgpu_gravity_amr_am_stats.restype = C.c_int
lib.tmgpu_gravity_amr_am_stats.argtypes = [_vp, C.POINTER(C.c_double)]
lib.tmgpu_gravity_amr_work.restype = C.c_int
lib.tmgpu_gravity_amr_work.argtypes = [_vp, _lp]
lib.tmgpu_gravity_amr_set_timing.restype = C.c_int
lib.tmgpu_gravity_amr_set_timing.argtypes = [_vp, C.c_int]
lib.tmgpu_gravity_amr_timing.restype = C.c_int
lib.tmgpu_gravity_amr_timing.argtypes = [_vp, C.POINTER(C.c_double), _lp]
lib.tmgpu_gravity_amr_distribute.restype = C.c_int
lib.tmgpu_gravity_amr_distribute.argtypes = [_vp, _vp, _lp, _ep]
lib.tmgpu_gravity_amr_set_peer.restype = C.c_int
lib.tmgpu_gravity_amr_set_peer.argtypes = [_vp, C.c_int, _ep]
lib.tmgpu_gravity_amr_mass_ptr.restype = _vp
lib.tmgpu_gravity_amr_mass_ptr.argtypes = [_vp]

GRAV_AM = 0x100


def _leaf_array(leaves):
    lv = np.ascontiguousarray(leaves, dtype=np.int32).reshape(-1, 4)
    return lv


def amr_plan_info(leaves):
    """Host-only plan build: (levels, nodes, W/X pairs, U-cross pairs)."""
    lv = _leaf_array(leaves)
    out = (C.c_longlong * 4)()
    err = TmgpuError()
    _lib.check(lib.tmgpu_gravity_amr_plan_info(lv.ctypes.data, lv.shape[0], out, C.byref(err)), err)
    return tuple(out)


lib.tmgpu_gravity_amr_plan_need.restype = C.c_int
lib.tmgpu_gravity_amr_plan_need.argtypes = [_vp, C.c_longlong, C.c_longlong, C.c_longlong, _lp,
                                            C.c_int, _ep]


def amr_plan_need(leaves, lo: int, hi: int):
    """Host-only: per-level counts of the patches whose M2L/L2L a rank owning
    the canonical slots [lo, hi) evaluates (the ancestors of its leaves)."""
    lv = _leaf_array(leaves)
    out = (C.c_longlong * 32)()
    err = TmgpuError()
    n = lib.tmgpu_gravity_amr_plan_need(lv.ctypes.data, lv.shape[0], lo, hi, out, 32, C.byref(err))
    if n < 0:
        _lib.check(-n, err)
    return list(out[:n])


lib.tmgpu_gravity_amr_let_plan.restype = C.c_int
lib.tmgpu_gravity_amr_let_plan.argtypes = [_vp, C.c_longlong, _lp, C.c_int, C.c_int, _lp, _lp, _lp, _lp,
                                           _lp, _ep]


def amr_let_plan(leaves, bounds, me: int):
    """Host-only: rank `me`'s multipole-moment exchange plan (csrc grav_let_plan):
    dict with owned/top/roots/halo_leaves counts and per-peer send/recv counts
    and list hashes."""
    lv = _leaf_array(leaves)
    b = np.ascontiguousarray(np.asarray(bounds, dtype=np.int64))
    world = len(b) - 1
    out = (C.c_longlong * 4)()
    arrs = [(C.c_longlong * world)() for _ in range(4)]
    err = TmgpuError()
    _lib.check(lib.tmgpu_gravity_amr_let_plan(lv.ctypes.data, lv.shape[0], b.ctypes.data_as(_lp), world,
                                              me, out, *arrs, C.byref(err)), err)
    return {"owned_internal": out[0], "top_internal": out[1], "roots": out[2], "halo_leaves": out[3],
            "send": list(arrs[0]), "recv": list(arrs[1]), "send_hash": list(arrs[2]),
            "recv_hash": list(arrs[3])}


def forest_leaf_array(forest):
    """[n, 4] (level, I, J, K) of a forest's local leaves in slot order."""
    from .amr import unpack

    return np.array([unpack(int(p)) for p in forest.local_leaves()], dtype=np.int32).reshape(-1, 4)


class GravityAMR:
    """Adaptive FMM over the cell tree of an octree forest (unit-cube root).

    leaves: [n, 4] (level, I, J, K) in canonical slot order (forest_leaf_array).
    Outputs are per leaf cell in slot order: phi[n*512], g[3, n*512]."""

    def __init__(self, leaves):
        self.leaves = _leaf_array(leaves)
        self.n = self.leaves.shape[0]
        err = TmgpuError()
        self.h = lib.tmgpu_gravity_amr_create(self.leaves.ctypes.data, self.n, C.byref(err))
        if not self.h:
            _lib.check(err.code or _lib.TMGPU_ERR_CUDA, err)

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:  # lib is None at interpreter exit
            lib.tmgpu_gravity_amr_destroy(self.h)
            self.h = None

    def info(self):
        out = (C.c_longlong * 4)()
        lib.tmgpu_gravity_amr_info(self.h, out)
        return tuple(out)

    def solve(self, mass=None, am=False, phi=None, g=None, stream=None, sync=True):
        """mass: numpy [n, 512] (host path, returns numpy) or CUDA tensor / None
        (device path: workspace masses when None; phi, g device tensors)."""
        flags = GRAV_AM if am else 0
        err = TmgpuError()
        ncell = self.local_cells()
        if isinstance(mass, np.ndarray):
            m = np.ascontiguousarray(mass, dtype=np.float64).reshape(-1)
            if m.size != ncell:
                raise ValueError("mass must have n*512 entries")
            phi_h, g_h = np.zeros(ncell), np.zeros(3 * ncell)
            _lib.check(lib.tmgpu_gravity_amr_solve(self.h, m.ctypes.data, phi_h.ctypes.data,
                                                   g_h.ctypes.data, flags | _lib.TMGPU_HOST_PTRS,
                                                   None, C.byref(err)), err)
            return phi_h, g_h.reshape(3, -1)
        import torch

        dev = mass.device if mass is not None else (phi.device if phi is not None else torch.device("cuda"))
        if phi is None:
            phi = torch.empty(ncell, dtype=torch.float64, device=dev)
        if g is None:
            g = torch.empty(3 * ncell, dtype=torch.float64, device=dev)
        st = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
        _lib.check(lib.tmgpu_gravity_amr_solve(self.h, None if mass is None else mass.data_ptr(),
                                               phi.data_ptr(), g.data_ptr(),
                                               flags | (0 if sync else _lib.TMGPU_ASYNC), st,
                                               C.byref(err)), err)
        return phi, g.view(3, -1)

    def mass_from_arena(self, forest, stream=None):
        err = TmgpuError()
        _lib.check(lib.tmgpu_gravity_amr_mass_from_arena(self.h, forest.arena_ptr(), forest.vars,
                                                         stream, C.byref(err)), err)

    def distribute(self, comm, owner) -> None:
        """Multi-GPU solve: this rank owns the canonical slots with
        owner[s] == comm.rank (contiguous ranges, partition_leaves). Masses
        (mass_from_arena / solve) and outputs become by local slot; the result
        equals the one-GPU solve bit for bit (csrc/gravity_amr.cu)."""
        o = np.asarray(owner)
        if len(o) != self.n:
            raise ValueError("owner must have one entry per leaf")
        if np.any(np.diff(o) < 0):
            raise ValueError("owner ranges must be contiguous and ascending")
        bounds = np.searchsorted(o, np.arange(comm.world + 1), side="left").astype(np.int64)
        bounds[-1] = self.n
        self._comm = comm
        self.lo, self.hi = int(bounds[comm.rank]), int(bounds[comm.rank + 1])
        err = TmgpuError()
        _lib.check(lib.tmgpu_gravity_amr_distribute(self.h, comm.h, bounds.ctypes.data_as(_lp),
                                                    C.byref(err)), err)

    def set_peer(self, on: bool = True) -> None:
        """Collective (after distribute): the moment exchange stores the subtree
        roots and halo patches straight into the peers' moment arrays (CUDA IPC
        over NVLink) instead of NCCL all-gather + send/recv; same bits."""
        err = TmgpuError()
        _lib.check(lib.tmgpu_gravity_amr_set_peer(self.h, 1 if on else 0, C.byref(err)), err)

    def local_cells(self) -> int:
        return (getattr(self, "hi", self.n) - getattr(self, "lo", 0)) * 512

    def work(self):
        """Algorithmic work of one solve: dict of interaction counts."""
        out = (C.c_longlong * 16)()
        lib.tmgpu_gravity_amr_work(self.h, out)
        kinds = ("ll", "li", "il", "ii")  # (target, source): l leaf, i internal
        return {"v_pairs": out[0], "wx_entries": out[1], "p2p_pairs": out[2],
                "u_cross_entries": out[3], "v_pairs_evaluated": out[4], "v_pairs_leaf": out[5],
                "wx_entries_leaf": out[6], **{"v_" + k: out[7 + q] for q, k in enumerate(kinds)},
                **{"wx_" + k: out[11 + q] for q, k in enumerate(kinds)}, "v_mono": out[15]}

    def set_timing(self, on: bool) -> None:
        lib.tmgpu_gravity_amr_set_timing(self.h, int(on))

    PHASES = ("up", "let", "m2l", "l2l", "l2p", "am", "k_mono", "k_fused", "k_wx")

    def timing(self):
        """(ms totals per phase, solves timed) since set_timing(True). k_mono,
        k_fused, k_wx: the M2L kernels alone (a timed solve serialises them)."""
        ms = (C.c_double * 9)()
        n = C.c_longlong()
        _lib.check(lib.tmgpu_gravity_amr_timing(self.h, ms, C.byref(n)), TmgpuError())
        return dict(zip(self.PHASES, ms)), n.value

    def am_stats(self):
        out = (C.c_double * 22)()
        lib.tmgpu_gravity_amr_am_stats(self.h, out)
        return np.array(out)
