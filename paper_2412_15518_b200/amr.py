"""AMR indexing, forest topology, device leaf arena and ghost exchange —
a mirror of the reference ``taskmesh::amr`` interface
(proj/include/taskmesh/amr/{morton,octree,ghost}.hpp) over libtmgpu.so.

Indexing (Morton keys, NodeId packing, canonical leaf order, face
neighbours, ghost-fill plans, partition_leaves) is host C++ and bit-exact
with the reference. Sub-grid state lives in a device arena
[slot][vars][S^3] (canonical leaf order); ``Forest.fill_ghosts`` runs the
reference-exact exchange (ghost.cpp:282-296) on the B200.
"""
from __future__ import annotations

import ctypes as C
import enum

import numpy as np

from . import _lib
from ._lib import TmgpuError, lib

_vp = C.c_void_p
_ep = C.POINTER(TmgpuError)
_u64p = C.POINTER(C.c_uint64)
_i64p = C.POINTER(C.c_int64)
_ip = C.POINTER(C.c_int)
_dp = C.POINTER(C.c_double)


def _sig(name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args


_sig("tmgpu_morton_encode", C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, _u64p, _ep])
_sig("tmgpu_morton_decode", C.c_int, [C.c_int, C.c_uint64, _u64p, _ep])
_sig("tmgpu_morton_dfs_rank", C.c_uint64, [C.c_int, C.c_uint64])
_sig("tmgpu_partition_leaves", C.c_int, [_u64p, C.c_size_t, C.c_int, _ip, _ep])
_sig("tmgpu_forest_create", _vp, [C.c_int, C.c_int, C.c_int, C.c_int, _ip, _ip, _ep])
_sig("tmgpu_forest_destroy", None, [_vp])
_sig("tmgpu_forest_refine", C.c_int, [_vp, C.c_uint64, _ep])
_sig("tmgpu_forest_coarsen", C.c_int, [_vp, C.c_uint64, _ep])
_sig("tmgpu_forest_regrid", C.c_int, [_vp, _u64p, C.c_size_t, _u64p, C.c_size_t, _ep])
_sig("tmgpu_forest_flag", C.c_int, [_vp, C.c_double, C.c_double, _ip, _ep])
_sig("tmgpu_forest_leaves", C.c_size_t, [_vp, _u64p, C.c_size_t])
_sig("tmgpu_forest_face_neighbor", C.c_int, [_vp, C.c_uint64, C.c_int, C.c_int, _u64p, _ip])
_sig("tmgpu_forest_plan", C.c_size_t, [_vp, C.c_int, _i64p, C.c_size_t])
_sig("tmgpu_forest_balanced", C.c_int, [_vp])
_sig("tmgpu_forest_cell_size", C.c_double, [_vp, C.c_int])
_sig("tmgpu_forest_topology_version", C.c_uint64, [_vp])
_sig("tmgpu_forest_exchanges", C.c_uint64, [_vp])
_sig("tmgpu_forest_scenario_refine", C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_double, _ep])
_sig("tmgpu_forest_scenario_fill", C.c_int, [_vp, C.c_int, C.c_uint64, _vp, _ep])
_sig("tmgpu_forest_alloc", C.c_int, [_vp, _ep])
_sig("tmgpu_forest_set_peer", C.c_int, [_vp, C.c_int, _ep])
_sig("tmgpu_forest_arena", _vp, [_vp])
_sig("tmgpu_forest_interior", C.c_int, [_vp, _vp, C.c_int, C.c_int, _vp, _ep])
_sig("tmgpu_forest_grids", C.c_int, [_vp, _vp, C.c_int, _ep])
_sig("tmgpu_forest_fill_ghosts", C.c_int, [_vp, _vp, _ep])
_sig("tmgpu_forest_fill_faces", C.c_int, [_vp, _vp, _ep])
_sig("tmgpu_forest_max_wavespeed", C.c_int, [_vp, C.c_double, _vp, _ep])
_sig("tmgpu_forest_step", C.c_int, [_vp, C.c_double, C.c_double, C.c_double, C.c_int, _vp, _dp,
                                    _ep])
_sig("tmgpu_forest_check", C.c_int, [_vp, _vp, _ep])
_sig("tmgpu_forest_distribute", C.c_int, [_vp, _vp, _ip, C.c_size_t, _ep])
_sig("tmgpu_forest_local_leaves", C.c_size_t, [_vp, _u64p, C.c_size_t])
_sig("tmgpu_forest_halo_manifest", C.c_size_t, [_vp, _ip, C.c_int, C.c_int, _i64p, C.c_size_t])
_sig("tmgpu_forest_floor_hits", C.c_int, [_vp, _vp, _ep])


class AmrError(ValueError):
    """Reference amr::AmrError (a std::logic_error)."""


def _amr_check(rc, err):
    if rc == _lib.TMGPU_ERR_AMR:
        raise AmrError(err.message.decode())
    _lib.check(rc, err)


# ------------------------------------------------------------------ morton / NodeId
def morton_encode(level: int, i: int, j: int, k: int) -> int:
    """morton.hpp:32-46 (returns the index of MortonKey{level, index})."""
    out = C.c_uint64(0)
    err = TmgpuError()
    _amr_check(lib.tmgpu_morton_encode(level, i, j, k, C.byref(out), C.byref(err)), err)
    return out.value


def morton_decode(level: int, index: int):
    out = (C.c_uint64 * 3)()
    err = TmgpuError()
    _amr_check(lib.tmgpu_morton_decode(level, index, out, C.byref(err)), err)
    return tuple(int(x) for x in out)


def morton_dfs_rank(level: int, index: int) -> int:
    return int(lib.tmgpu_morton_dfs_rank(level, index))


def pack(level: int, ci: int, cj: int, ck: int) -> int:
    """NodeId::packed (octree.hpp:29-33)."""
    return (level << 60) | (ci << 40) | (cj << 20) | ck


def unpack(p: int):
    p = int(p)
    return p >> 60, (p >> 40) & 0xFFFFF, (p >> 20) & 0xFFFFF, p & 0xFFFFF


def partition_leaves(weights, localities: int) -> list[int]:
    """octree.cpp:374-399: greedy contiguous cut, ranges never empty."""
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.uint64))
    owner = np.zeros(len(w), dtype=np.int32)
    err = TmgpuError()
    rc = lib.tmgpu_partition_leaves(w.ctypes.data_as(_u64p), len(w), localities,
                                    owner.ctypes.data_as(_ip), C.byref(err))
    _amr_check(rc, err)
    return owner.tolist()


class NeighborKind(enum.IntEnum):
    same = 0
    coarser = 1
    finer = 2
    boundary = 3


class Boundary(enum.IntEnum):
    periodic = 0
    reflective = 1


class Scenario(enum.IntEnum):
    rotating_star = 0
    double_white_dwarf = 1
    sod = 2
    sedov = 3


class Forest:
    """The reference amr::Tree (octree.hpp:241-314) with grids in device memory."""

    def __init__(self, edge=8, ghost=2, vars=5, max_level=10, root_dims=(1, 1, 1),
                 bc=(0, 0, 0)):
        err = TmgpuError()
        self.edge, self.ghost, self.vars, self.max_level = edge, ghost, vars, max_level
        self.stride = edge + 2 * ghost
        self.root_dims, self.bc = tuple(root_dims), tuple(int(b) for b in bc)
        self.h = lib.tmgpu_forest_create(edge, ghost, vars, max_level, (C.c_int * 3)(*root_dims),
                                         (C.c_int * 3)(*self.bc), C.byref(err))
        if not self.h:
            raise AmrError(err.message.decode())

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:  # lib is None at interpreter exit
            lib.tmgpu_forest_destroy(self.h)
            self.h = None

    # -- topology (host, bit-exact)
    def refine(self, node) -> None:
        err = TmgpuError()
        _amr_check(lib.tmgpu_forest_refine(self.h, int(node), C.byref(err)), err)

    def coarsen(self, node) -> None:
        """Tree::coarsen (octree.cpp:236-293), topology only."""
        err = TmgpuError()
        _amr_check(lib.tmgpu_forest_coarsen(self.h, int(node), C.byref(err)), err)

    def regrid(self, refine=(), coarsen=()) -> None:
        """Refine then coarsen with the device data carried along exactly as the
        reference's Tree::refine / coarsen carry their grids (prolong_cell /
        restrict_cells, octree.cpp:149-293); the arena is rebuilt. Single GPU."""
        r = np.ascontiguousarray(np.asarray(refine, dtype=np.uint64))
        c = np.ascontiguousarray(np.asarray(coarsen, dtype=np.uint64))
        err = TmgpuError()
        _amr_check(lib.tmgpu_forest_regrid(self.h, r.ctypes.data_as(_u64p), len(r),
                                           c.ctypes.data_as(_u64p), len(c), C.byref(err)), err)

    def flag_refinement(self, theta: float, rho_floor: float = 1e-10) -> np.ndarray:
        """Tree::flag_refinement (octree.cpp:295-323) of every local leaf on the
        device state (ghosts as they are): bool per slot."""
        out = np.zeros(self.local_count(), dtype=np.int32)
        err = TmgpuError()
        _lib.check(lib.tmgpu_forest_flag(self.h, theta, rho_floor, out.ctypes.data_as(_ip),
                                         C.byref(err)), err)
        return out.astype(bool)

    def leaves(self) -> np.ndarray:
        n = lib.tmgpu_forest_leaves(self.h, None, 0)
        out = np.zeros(n, dtype=np.uint64)
        lib.tmgpu_forest_leaves(self.h, out.ctypes.data_as(_u64p), n)
        return out

    def is_leaf(self, node) -> bool:
        lib.tmgpu_forest_is_leaf.restype = C.c_int
        lib.tmgpu_forest_is_leaf.argtypes = [C.c_void_p, C.c_uint64]
        return bool(lib.tmgpu_forest_is_leaf(self.h, int(node)))

    def leaf_count(self) -> int:
        return int(lib.tmgpu_forest_leaves(self.h, None, 0))

    def face_neighbor(self, leaf, axis: int, direction: int):
        ids = np.zeros(4, dtype=np.uint64)
        cnt = C.c_int(0)
        kind = lib.tmgpu_forest_face_neighbor(self.h, int(leaf), axis, direction,
                                              ids.ctypes.data_as(_u64p), C.byref(cnt))
        if kind < 0:
            raise AmrError("face_neighbor: topology corrupt")
        return NeighborKind(kind), [int(x) for x in ids[: cnt.value]]

    def plan(self, axis: int) -> np.ndarray:
        n = lib.tmgpu_forest_plan(self.h, axis, None, 0)
        rows = np.zeros((n, 7), dtype=np.int64)
        lib.tmgpu_forest_plan(self.h, axis, rows.ctypes.data_as(_i64p), n)
        return rows

    def is_balanced(self) -> bool:
        return bool(lib.tmgpu_forest_balanced(self.h))

    def cell_size(self, level: int) -> float:
        return float(lib.tmgpu_forest_cell_size(self.h, level))

    def topology_version(self) -> int:
        return int(lib.tmgpu_forest_topology_version(self.h))

    def exchanges(self) -> int:
        return int(lib.tmgpu_forest_exchanges(self.h))

    def scenario_refine(self, kind: Scenario, min_level: int, max_level: int,
                        theta: float = 0.1) -> None:
        err = TmgpuError()
        _amr_check(lib.tmgpu_forest_scenario_refine(self.h, int(kind), min_level, max_level, theta,
                                                    C.byref(err)), err)

    def scenario_state(self, kind: Scenario, seed: int = 2412518) -> np.ndarray:
        """Initial interior state, compact [slot][vars][E^3] float64 (host)."""
        out = np.zeros((self.leaf_count(), self.vars, self.edge ** 3))
        err = TmgpuError()
        _lib.check(lib.tmgpu_forest_scenario_fill(self.h, int(kind), seed, out.ctypes.data,
                                                  C.byref(err)), err)
        return out

    # -- distribution (one process per GPU)
    def distribute(self, comm, owner) -> None:
        """Own the leaves with owner[g] == comm.rank (partition_leaves over the
        canonical order); the device arena then holds only local leaves."""
        o = np.ascontiguousarray(np.asarray(owner, dtype=np.int32))
        err = TmgpuError()
        self._comm = comm  # keep the communicator alive as long as the forest
        self._owner = o
        _lib.check(lib.tmgpu_forest_distribute(self.h, comm.h if comm else None,
                                               o.ctypes.data_as(_ip), len(o), C.byref(err)), err)

    def local_leaves(self) -> np.ndarray:
        n = lib.tmgpu_forest_local_leaves(self.h, None, 0)
        out = np.zeros(n, dtype=np.uint64)
        lib.tmgpu_forest_local_leaves(self.h, out.ctypes.data_as(_u64p), n)
        return out

    def local_count(self) -> int:
        return int(lib.tmgpu_forest_local_leaves(self.h, None, 0))

    def halo_manifest(self, owner, rank: int, world: int) -> np.ndarray:
        """Host-only: every slab rank `rank` sends/receives per exchange, rows
        (send 0 | recv 1, peer, dst leaf, src leaf, kind, axis, dir)."""
        o = np.ascontiguousarray(np.asarray(owner, dtype=np.int32))
        n = lib.tmgpu_forest_halo_manifest(self.h, o.ctypes.data_as(_ip), rank, world, None, 0)
        rows = np.zeros((n, 7), dtype=np.int64)
        lib.tmgpu_forest_halo_manifest(self.h, o.ctypes.data_as(_ip), rank, world,
                                       rows.ctypes.data_as(_i64p), n)
        return rows

    # -- device state
    def alloc(self) -> None:
        """(Re)allocate the zeroed device arena for the current topology."""
        err = TmgpuError()
        _lib.check(lib.tmgpu_forest_alloc(self.h, C.byref(err)), err)

    def set_peer(self, on: bool = True) -> None:
        """Collective: move the cross-GPU ghost slabs through peer memory (CUDA
        IPC over NVLink) instead of NCCL send/recv; re-call after alloc()."""
        err = TmgpuError()
        _lib.check(lib.tmgpu_forest_set_peer(self.h, 1 if on else 0, C.byref(err)), err)
        self._peer = bool(on)

    def arena_ptr(self) -> int:
        return int(lib.tmgpu_forest_arena(self.h) or 0)

    def set_interior(self, compact, stream=None, sync: bool = True) -> None:
        """Interior state [local leaves][V][E^3] into the arena (host or device
        buffer). stream/sync=False: enqueue on that stream and return."""
        self._interior(compact, True, stream, sync)

    def get_interior(self, out=None, stream=None, sync: bool = True):
        if out is None:
            out = np.zeros((self.local_count(), self.vars, self.edge ** 3))
        self._interior(out, False, stream, sync)
        return out

    def _interior(self, buf, to_device, stream=None, sync=True):
        from .hydro import _addr

        ptr, host, st, n = _addr(buf)
        if n != self.local_count() * self.vars * self.edge ** 3:
            raise ValueError("compact interior has the wrong size")
        if stream is not None:
            st = stream
        flags = (_lib.TMGPU_HOST_PTRS if host else 0) | (0 if sync else _lib.TMGPU_ASYNC)
        err = TmgpuError()
        _lib.check(lib.tmgpu_forest_interior(self.h, ptr, 1 if to_device else 0, flags, st,
                                             C.byref(err)), err)

    def get_grids(self) -> np.ndarray:
        out = np.zeros((self.local_count(), self.vars * self.stride ** 3))
        err = TmgpuError()
        _lib.check(lib.tmgpu_forest_grids(self.h, out.ctypes.data, 0, C.byref(err)), err)
        return out

    def set_grids(self, grids: np.ndarray) -> None:
        g = np.ascontiguousarray(grids, dtype=np.float64)
        err = TmgpuError()
        _lib.check(lib.tmgpu_forest_grids(self.h, g.ctypes.data, 1, C.byref(err)), err)

    def arena_grids(self, which: int, grids=None, out=None):
        """Whole ghosted blocks [local][V*S^3] of the current (which=0) or the
        other ping-pong arena (which=1); with `grids`, write them instead.
        `grids` / `out` may also be CUDA tensors (device-to-device copy)."""
        lib.tmgpu_forest_arena_grids.restype = C.c_int
        lib.tmgpu_forest_arena_grids.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                                                 C.POINTER(TmgpuError)]
        err = TmgpuError()
        n = self.local_count() * self.vars * self.stride ** 3
        if grids is None:
            if out is None:
                out = np.zeros((self.local_count(), self.vars * self.stride ** 3))
            ptr = out.data_ptr() if hasattr(out, "data_ptr") else out.ctypes.data
            if (out.numel() if hasattr(out, "numel") else out.size) != n:
                raise ValueError("out must hold every local leaf's ghosted block")
            _lib.check(lib.tmgpu_forest_arena_grids(self.h, which, ptr, 0, C.byref(err)), err)
            return out
        if hasattr(grids, "data_ptr"):  # CUDA tensor
            if grids.numel() != n or not grids.is_contiguous():
                raise ValueError("grids must be a contiguous block of every local leaf")
            _lib.check(lib.tmgpu_forest_arena_grids(self.h, which, grids.data_ptr(), 1, C.byref(err)), err)
            return None
        g = np.ascontiguousarray(grids, dtype=np.float64)
        if g.size != self.local_count() * self.vars * self.stride ** 3:
            raise ValueError("grids must hold every local leaf's ghosted block")
        _lib.check(lib.tmgpu_forest_arena_grids(self.h, which, g.ctypes.data, 1, C.byref(err)), err)
        return None

    def fill_ghosts(self, stream=None) -> None:
        """ghost::fill_ghosts_sync (ghost.cpp:282-296) on the device."""
        err = TmgpuError()
        _lib.check(lib.tmgpu_forest_fill_ghosts(self.h, stream, C.byref(err)), err)

    def fill_faces(self, stream=None) -> None:
        """One-round face-only exchange (the step's default): every ghost the
        stage reads, bitwise equal to fill_ghosts_sync; edges/corners untouched."""
        err = TmgpuError()
        _lib.check(lib.tmgpu_forest_fill_faces(self.h, stream, C.byref(err)), err)

    def max_wavespeed(self, gamma: float = 1.4) -> np.ndarray:
        out = np.zeros(self.local_count())
        err = TmgpuError()
        _lib.check(lib.tmgpu_forest_max_wavespeed(self.h, gamma, out.ctypes.data, C.byref(err)),
                   err)
        return out

    def floor_hits(self) -> np.ndarray:
        out = np.zeros(self.local_count())
        err = TmgpuError()
        _lib.check(lib.tmgpu_forest_floor_hits(self.h, out.ctypes.data, C.byref(err)), err)
        return out


def build_scenario(kind: Scenario, min_level: int, max_level: int, theta: float = 0.1,
                   bc=(0, 0, 0), root_dims=(1, 1, 1)) -> Forest:
    f = Forest(vars=5, max_level=max_level, bc=bc, root_dims=root_dims)
    f.scenario_refine(kind, min_level, max_level, theta)
    return f
