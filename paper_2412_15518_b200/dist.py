"""Leaf-to-GPU distribution: one process per GPU, leaves partitioned with the
reference's partition_leaves (octree.cpp:374-399) over the canonical leaf
order, ghost slabs crossing GPUs moved by grouped NCCL send/recv inside the
step (csrc/comm.cpp, csrc/halo_plan.cpp), the CFL dt min-reduced with
ncclAllReduce. torch.distributed is used only to broadcast the NCCL id.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import TmgpuError, lib
from .amr import Forest, partition_leaves

_vp = C.c_void_p
_ep = C.POINTER(TmgpuError)
lib.tmgpu_comm_unique_id.restype = C.c_int
lib.tmgpu_comm_unique_id.argtypes = [C.c_char_p, _ep]
lib.tmgpu_comm_create.restype = _vp
lib.tmgpu_comm_create.argtypes = [C.c_int, C.c_int, C.c_char_p, _ep]
lib.tmgpu_comm_destroy.restype = None
lib.tmgpu_comm_destroy.argtypes = [_vp]


class Comm:
    """NCCL communicator over the ranks of the default torch process group."""

    def __init__(self, rank: int, world: int, unique_id: bytes):
        err = TmgpuError()
        self.rank, self.world = rank, world
        self.h = lib.tmgpu_comm_create(rank, world, unique_id, C.byref(err))
        if not self.h:
            _lib.check(err.code or _lib.TMGPU_ERR_CUDA, err)

    @staticmethod
    def from_torch() -> "Comm":
        import torch
        import torch.distributed as dist

        rank, world = dist.get_rank(), dist.get_world_size()
        buf = C.create_string_buffer(128)
        if rank == 0:
            err = TmgpuError()
            _lib.check(lib.tmgpu_comm_unique_id(buf, C.byref(err)), err)
        t = torch.tensor(list(buf.raw), dtype=torch.uint8,
                         device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.broadcast(t, 0)
        return Comm(rank, world, bytes(t.cpu().tolist()))

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:  # lib is None at interpreter exit
            lib.tmgpu_comm_destroy(self.h)
            self.h = None


def partition(forest: Forest, world: int, weights=None) -> list[int]:
    """Owner rank per canonical leaf: partition_leaves with 512 per leaf
    (cells per sub-grid) unless weights are given."""
    n = forest.leaf_count()
    w = np.full(n, forest.edge ** 3, dtype=np.uint64) if weights is None else weights
    return partition_leaves(w, world)


def local_range(owner, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) of the canonical leaves owned by `rank`."""
    o = np.asarray(owner)
    idx = np.nonzero(o == rank)[0]
    return (int(idx[0]), int(idx[-1]) + 1) if len(idx) else (0, 0)
