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


def replay_topology(forest: Forest, leaves) -> Forest:
    """A one-GPU Forest with the same configuration and leaves (the internal
    nodes refined in level order; a node a 2:1 cascade already refined is skipped)."""
    from .amr import pack, unpack

    g = Forest(forest.edge, forest.ghost, forest.vars, forest.max_level, forest.root_dims, forest.bc)
    internal = set()
    for p in leaves:
        lvl, ci, cj, ck = unpack(int(p))
        for l in range(lvl):
            sh = lvl - l
            internal.add(pack(l, ci >> sh, cj >> sh, ck >> sh))
    for p in sorted(internal, key=lambda q: (q >> 60, q)):
        if g.is_leaf(p):
            g.refine(p)
    if not np.array_equal(g.leaves(), np.asarray(leaves, dtype=np.uint64)):
        raise RuntimeError("replayed topology differs")
    return g


def regrid(forest: Forest, refine=(), coarsen=(), weights=None) -> None:
    """Collective AMR regrid of a distributed forest (every rank passes the same
    lists): refine then coarsen with the state carried along exactly as the
    one-GPU Forest.regrid (the reference's prolong_cell / restrict_cells,
    octree.cpp:149-293), then re-partition the new leaves (partition_leaves) and
    move every block to its new owner.

    The data path funnels through rank 0 over NVLink: the ranks' ghosted blocks
    are gathered there, the one-GPU regrid runs on the whole arena (so the
    result is the one-GPU result, bit for bit), and the new blocks are sent to
    their owners. A regrid is a rare topology change; at configs[4] (15.8 GB of
    blocks) the gather and scatter are tens of ms at NVLink rates. The forest's
    peer-memory exchange, when on, is rebuilt for the new distribution.
    Prolongation reads the parent's face ghosts as they are (like the reference's
    Tree::refine): the drivers' regrid fills every face ghost first
    (Forest.fill_faces), which makes the distributed and one-GPU inputs equal."""
    import torch
    import torch.distributed as tdist

    comm = forest._comm
    rank, world = comm.rank, comm.world
    blk = forest.vars * forest.stride ** 3
    old_owner = np.asarray(forest._owner)
    peer = getattr(forest, "_peer", False)
    if peer:
        forest.set_peer(False)  # collective
    dev = torch.device("cuda", torch.cuda.current_device())
    mine = torch.empty(forest.local_count() * blk, dtype=torch.float64, device=dev)
    forest.arena_grids(0, out=mine)
    counts = np.bincount(old_owner, minlength=world)
    full = None
    if rank == 0:
        full = torch.empty(int(counts.sum()) * blk, dtype=torch.float64, device=dev)
        off = np.concatenate([[0], np.cumsum(counts)]) * blk
        full[off[0]:off[1]].copy_(mine)
        reqs = [tdist.irecv(full[off[q]:off[q + 1]], src=q) for q in range(1, world) if counts[q]]
        for r in reqs:
            r.wait()
    elif len(mine):
        tdist.send(mine, dst=0)
    refine = [int(x) for x in refine]
    coarsen = [int(x) for x in coarsen]
    new_blocks = None
    if rank == 0:
        g = replay_topology(forest, forest.leaves())
        g.alloc()
        g.arena_grids(0, full)
        del full
        g.regrid(refine, coarsen)
        new_blocks = torch.empty(g.leaf_count() * blk, dtype=torch.float64, device=dev)
        g.arena_grids(0, out=new_blocks)
        del g
    for r in refine:  # the same topology change on every rank (deterministic cascades)
        forest.refine(r)
    for c in coarsen:
        forest.coarsen(c)
    owner = partition(forest, world, weights)
    forest.distribute(comm, owner)
    forest.alloc()
    counts = np.bincount(np.asarray(owner), minlength=world)
    got = torch.empty(forest.local_count() * blk, dtype=torch.float64, device=dev)
    if rank == 0:
        off = np.concatenate([[0], np.cumsum(counts)]) * blk
        got.copy_(new_blocks[off[0]:off[1]])
        reqs = [tdist.isend(new_blocks[off[q]:off[q + 1]], dst=q) for q in range(1, world) if counts[q]]
        for r in reqs:
            r.wait()
    elif len(got):
        tdist.recv(got, src=0)
    torch.cuda.synchronize()
    forest.arena_grids(0, got)
    if peer:
        forest.set_peer(True)  # collective
