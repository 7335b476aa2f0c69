"""Checkpoint files: the reference's specified state dump ("flat binary
of (key, cell payload) records, little-endian, versioned header — used for bitwise
equivalence tests across backends"; a run writes one after its
steps, and identical config + seed give identical bytes). The reference specifies
the format but ships no writer, so the layout below is ours:

    header (40 bytes, little-endian)
        magic     4s   b"TMCK"
        version   u8   2 (version-1 files, identical but without the ghost byte, load too)
        flags     u8   bit 0: RESUMABLE (ghosted payload, below)
        vars      u16  conserved variables per cell (5 Euler, 1 scalar)
        edge      u16  sub-grid edge E (8)
        ghost     u8   ghost layers G (2; 0 in version-1 files)
        reserved  5 bytes, zero
        time      f64  simulation time
        step      u64  completed steps
        records   u64  number of records
    records, in canonical leaf order (root raster, then Morton DFS — the order of
    Forest.leaves(), octree.cpp:52-77)
        key       u64  packed NodeId of the leaf (amr.pack; octree.hpp:23-49)
        payload   f64[vars][E^3]  interior cells, x fastest (the compact layout of
                  Forest.get_interior), or with RESUMABLE
                  f64[2][vars][S^3]  the whole ghosted blocks of the current and the
                  other ping-pong arena (S = E + 2G): the step carries both arenas'
                  ghost layers across exchanges, so only these let a resumed run
                  continue bit for bit (tests/test_checkpoint.py)

With several ranks (partition_leaves ranges are contiguous in canonical order)
every rank writes its own records' byte range of the file; rank 0 writes the
header first. Nothing is gathered, so a partitioned run and a one-GPU run of the
same step produce the same bytes without any rank holding the whole state.
"""
from __future__ import annotations

import os
import struct

import numpy as np

MAGIC = b"TMCK"
VERSION = 2
RESUMABLE = 0x1
_HEADER = struct.Struct("<4sBBHHB5xdQQ")
HEADER_BYTES = _HEADER.size  # 40


class CheckpointError(ValueError):
    pass


def _record_dtype(vars_: int, edge: int, ghost: int, flags: int) -> np.dtype:
    n = 2 * vars_ * (edge + 2 * ghost) ** 3 if flags & RESUMABLE else vars_ * edge ** 3
    return np.dtype([("key", "<u8"), ("payload", "<f8", (n,))])


def encode(keys, payload, time: float = 0.0, step: int = 0, ghost: int | None = None,
           flags: int = 0) -> bytes:
    """Serialise records: keys [n] (uint64 packed NodeIds), payload [n][vars][E^3]
    (or with flags=RESUMABLE, [n][2][vars][S^3] and the ghost width)."""
    keys = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64))
    payload = np.asarray(payload, dtype=np.float64)
    n = keys.shape[0]
    if payload.shape[0] != n:
        raise CheckpointError(f"payload shape {payload.shape} does not match {n} keys")
    if flags & RESUMABLE:
        if payload.ndim != 4 or payload.shape[1] != 2 or ghost is None:
            raise CheckpointError("a resumable payload is [n][2][vars][S^3] with the ghost width")
        vars_, S = payload.shape[2], round(payload.shape[3] ** (1.0 / 3.0))
        edge = S - 2 * ghost
        if S ** 3 != payload.shape[3] or edge <= 0:
            raise CheckpointError(f"{payload.shape[3]} cells per block is not a ghosted cube")
    else:
        if payload.ndim != 3:
            raise CheckpointError(f"payload shape {payload.shape} does not match {n} keys")
        vars_, cells = payload.shape[1], payload.shape[2]
        edge = round(cells ** (1.0 / 3.0))
        if edge ** 3 != cells:
            raise CheckpointError(f"{cells} cells per record is not a cube")
        ghost = ghost or 0
    rec = np.empty(n, dtype=_record_dtype(vars_, edge, ghost, flags))
    rec["key"] = keys
    rec["payload"] = payload.reshape(n, rec.dtype["payload"].shape[0])
    return header(vars_, edge, ghost, n, time, step, flags) + rec.tobytes()


def header(vars_: int, edge: int, ghost: int, n: int, time: float, step: int, flags: int = 0) -> bytes:
    return _HEADER.pack(MAGIC, VERSION, flags, vars_, edge, ghost, float(time), int(step), n)


def _parse_header(buf) -> dict:
    if len(buf) < HEADER_BYTES:
        raise CheckpointError("truncated checkpoint header")
    magic, version, flags, vars_, edge, ghost, time, step, n = _HEADER.unpack_from(bytes(buf[:HEADER_BYTES]), 0)
    if magic != MAGIC:
        raise CheckpointError(f"not a checkpoint (magic {magic!r})")
    if version not in (1, 2):
        raise CheckpointError(f"unsupported checkpoint version {version}")
    if version == 1:
        ghost, flags = 0, 0
    return {"version": version, "flags": flags, "vars": vars_, "edge": edge, "ghost": ghost,
            "time": time, "step": step, "records": n}


def decode(buf):
    """-> (header dict, keys [n] uint64, payload [n][vars][E^3] float64, or
    [n][2][vars][S^3] for a RESUMABLE file)."""
    head = _parse_header(buf)
    dt = _record_dtype(head["vars"], head["edge"], head["ghost"], head["flags"])
    n = head["records"]
    if len(buf) != HEADER_BYTES + n * dt.itemsize:
        raise CheckpointError(f"checkpoint holds {len(buf) - HEADER_BYTES} record bytes, "
                              f"expected {n * dt.itemsize}")
    rec = np.frombuffer(buf, dtype=dt, count=n, offset=HEADER_BYTES)
    cells = (head["edge"] + 2 * head["ghost"]) ** 3 if head["flags"] & RESUMABLE else head["edge"] ** 3
    shape = ((n, 2, head["vars"], cells) if head["flags"] & RESUMABLE else (n, head["vars"], cells))
    return head, rec["key"].astype(np.uint64), rec["payload"].astype(np.float64).reshape(shape)


def merge(order, parts):
    """Records of several ranks [(keys, payload), ...] into the canonical order
    `order` (Forest.leaves()); every key must appear exactly once."""
    order = np.asarray(order, dtype=np.uint64)
    pos = {int(k): i for i, k in enumerate(order)}
    first = next((np.asarray(p) for _, p in parts if len(p)), None)
    if first is None:
        if len(order):
            raise CheckpointError(f"{len(order)} leaves missing from the merged records")
        return order, np.zeros((0,) + tuple(np.asarray(parts[0][1]).shape[1:]) if parts else (0,))
    out = np.empty((len(order),) + first.shape[1:], dtype=np.float64)
    seen = np.zeros(len(order), dtype=bool)
    for keys, payload in parts:
        for k, row in zip(np.asarray(keys, dtype=np.uint64), np.asarray(payload)):
            i = pos.get(int(k))
            if i is None or seen[i]:
                raise CheckpointError(f"leaf {int(k):#x} unknown or contributed twice")
            seen[i] = True
            out[i] = row
    if not seen.all():
        raise CheckpointError(f"{int((~seen).sum())} leaves missing from the merged records")
    return order, out


def _world(group):
    try:
        import torch.distributed as tdist
    except ImportError:  # pragma: no cover
        return None, 1, 0
    if tdist.is_available() and tdist.is_initialized() and tdist.get_world_size(group) > 1:
        return tdist, tdist.get_world_size(group), tdist.get_rank(group)
    return None, 1, 0


def _local_payload(forest, state, resumable, stream):
    if resumable:
        if state is not None:
            raise CheckpointError("a resumable checkpoint is taken from the device arenas")
        blocks = [forest.arena_grids(w) for w in (0, 1)]  # synchronises the device
        return np.stack(blocks, axis=1).reshape(forest.local_count(), 2, forest.vars, -1)
    if state is not None:
        return np.asarray(state, dtype=np.float64)
    return forest.get_interior(stream=stream)


def save(path, forest, time: float = 0.0, step: int = 0, state=None, keys=None,
         group=None, resumable: bool = False, stream=None) -> bytes | None:
    """Write the forest's state: the device arena's interiors (or `state`
    [local][V][E^3] for the leaves `keys`, default this rank's leaves), or with
    `resumable` both arenas' ghosted blocks (bitwise restart). `stream`: the
    CUDA stream the steps were enqueued on (read after them).

    Collective with more than one torch.distributed rank. With a `path` every
    rank writes its own contiguous byte range (rank 0 the header first) and
    nothing is gathered; returns None. Without a path the records are gathered on
    rank 0, which returns the merged bytes (None elsewhere). Single process:
    returns the bytes."""
    tdist, world, rank = _world(group)
    local = _local_payload(forest, state, resumable, stream)
    keys = forest.local_leaves() if keys is None else keys
    keys = np.asarray(keys, dtype=np.uint64)
    flags = RESUMABLE if resumable else 0
    ghost = forest.ghost if resumable else 0
    if tdist is None:
        buf = encode(keys, local, time, step, ghost=ghost, flags=flags)
        if path is not None:
            with open(path, "wb") as fh:
                fh.write(buf)
        return buf
    order = np.asarray(forest.leaves(), dtype=np.uint64)
    if path is None:  # in-memory: gather to rank 0 only
        parts = [None] * world if rank == 0 else None
        tdist.gather_object((keys, local), parts, dst=0, group=group)
        if rank != 0:
            return None
        keys_all, full = merge(order, parts)
        return encode(keys_all, full, time, step, ghost=ghost, flags=flags)
    pos = {int(k): i for i, k in enumerate(order)}
    idx = np.array([pos.get(int(k), -1) for k in keys], dtype=np.int64)
    if len(idx) and ((idx < 0).any() or (np.diff(idx) != 1).any()):
        raise CheckpointError("a rank's leaves must be a contiguous range of the canonical order")
    dt = _record_dtype(forest.vars, forest.edge, ghost, flags)
    if rank == 0:
        with open(path, "wb") as fh:
            fh.write(header(forest.vars, forest.edge, ghost, len(order), time, step, flags))
            fh.truncate(HEADER_BYTES + len(order) * dt.itemsize)
    tdist.barrier(group=group)
    if len(idx):
        rec = np.empty(len(idx), dtype=dt)
        rec["key"] = keys
        rec["payload"] = local.reshape(len(idx), dt["payload"].shape[0])
        with open(path, "r+b") as fh:
            fh.seek(HEADER_BYTES + int(idx[0]) * dt.itemsize)
            fh.write(rec.tobytes())
    tdist.barrier(group=group)
    return None


def load(path, forest, stream=None):
    """Read a checkpoint into the forest's device arena(s) (this rank's leaves,
    read from the file's mapped records): the records must cover the forest's
    leaves exactly. A RESUMABLE file restores both arenas' ghosted blocks, so
    stepping on continues bit for bit. Returns the header."""
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        head = _parse_header(fh.read(HEADER_BYTES))
    if head["vars"] != forest.vars or head["edge"] != forest.edge:
        raise CheckpointError(f"checkpoint is V={head['vars']} E={head['edge']}, forest "
                              f"V={forest.vars} E={forest.edge}")
    dt = _record_dtype(head["vars"], head["edge"], head["ghost"], head["flags"])
    n = head["records"]
    if size != HEADER_BYTES + n * dt.itemsize:
        raise CheckpointError(f"checkpoint holds {size - HEADER_BYTES} record bytes, "
                              f"expected {n * dt.itemsize}")
    order = np.asarray(forest.leaves(), dtype=np.uint64)
    if n != len(order):
        raise CheckpointError(f"checkpoint has {n} records, the forest {len(order)} leaves")
    rec = np.memmap(path, dtype=dt, mode="r", offset=HEADER_BYTES, shape=(n,)) if n else np.zeros(0, dt)
    if n and not np.array_equal(np.asarray(rec["key"]), order):
        merge(order, [(np.asarray(rec["key"]), np.zeros((n, 1)))])  # names the culprit
        raise CheckpointError("records are not in the forest's canonical leaf order")
    pos = {int(k): i for i, k in enumerate(order)}
    mine = np.array([pos[int(k)] for k in forest.local_leaves()], dtype=np.int64)
    local = np.asarray(rec["payload"][mine]) if n else np.zeros((0, dt["payload"].shape[0]))
    if head["flags"] & RESUMABLE:
        if head["ghost"] != forest.ghost:
            raise CheckpointError(f"checkpoint ghost width {head['ghost']}, forest {forest.ghost}")
        blocks = local.reshape(len(mine), 2, -1)
        for w in (0, 1):
            forest.arena_grids(w, np.ascontiguousarray(blocks[:, w]))
    else:
        forest.set_interior(np.ascontiguousarray(local.reshape(len(mine), forest.vars, -1)), stream=stream)
    return head
