"""Checkpoint files: the reference's specified state dump ("flat binary
of (key, cell payload) records, little-endian, versioned header — used for bitwise
equivalence tests across backends"; a run writes one after its
steps, and identical config + seed give identical bytes). The reference specifies
the format but ships no writer, so the layout below is ours:

    header (40 bytes, little-endian)
        magic     4s   b"TMCK"
        version   u8   1
        flags     u8   0 (reserved)
        vars      u16  conserved variables per cell (5 Euler, 1 scalar)
        edge      u16  sub-grid edge E (8)
        reserved  6 bytes, zero
        time      f64  simulation time
        step      u64  completed steps
        records   u64  number of records
    records, in canonical leaf order (root raster, then Morton DFS — the order of
    Forest.leaves(), octree.cpp:52-77)
        key       u64  packed NodeId of the leaf (amr.pack; octree.hpp:23-49)
        payload   f64[vars][E^3]  interior cells, x fastest (the compact layout of
                  Forest.get_interior)

Host-side I/O only: the state comes off the device through Forest.get_interior.
With several ranks every rank contributes its local leaves and rank 0 writes the
merged file, so a partitioned run and a one-GPU run of the same step produce the
same bytes.
"""
from __future__ import annotations

import struct

import numpy as np

MAGIC = b"TMCK"
VERSION = 1
_HEADER = struct.Struct("<4sBBHH6xdQQ")
HEADER_BYTES = _HEADER.size  # 40


class CheckpointError(ValueError):
    pass


def encode(keys, payload, time: float = 0.0, step: int = 0) -> bytes:
    """Serialise records: keys [n] (uint64 packed NodeIds), payload [n][vars][E^3]."""
    keys = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64))
    payload = np.asarray(payload, dtype=np.float64)
    if payload.ndim != 3 or payload.shape[0] != keys.shape[0]:
        raise CheckpointError(f"payload shape {payload.shape} does not match {keys.shape[0]} keys")
    n, vars_, cells = payload.shape
    edge = round(cells ** (1.0 / 3.0))
    if edge ** 3 != cells:
        raise CheckpointError(f"{cells} cells per record is not a cube")
    rec = np.empty(n, dtype=np.dtype([("key", "<u8"), ("payload", "<f8", (vars_ * cells,))]))
    rec["key"] = keys
    rec["payload"] = payload.reshape(n, vars_ * cells)
    head = _HEADER.pack(MAGIC, VERSION, 0, vars_, edge, float(time), int(step), n)
    return head + rec.tobytes()


def decode(buf: bytes):
    """-> (header dict, keys [n] uint64, payload [n][vars][E^3] float64)."""
    if len(buf) < HEADER_BYTES:
        raise CheckpointError("truncated checkpoint header")
    magic, version, flags, vars_, edge, time, step, n = _HEADER.unpack_from(buf, 0)
    if magic != MAGIC:
        raise CheckpointError(f"not a checkpoint (magic {magic!r})")
    if version != VERSION:
        raise CheckpointError(f"unsupported checkpoint version {version}")
    cells = edge ** 3
    dt = np.dtype([("key", "<u8"), ("payload", "<f8", (vars_ * cells,))])
    if len(buf) != HEADER_BYTES + n * dt.itemsize:
        raise CheckpointError(f"checkpoint holds {len(buf) - HEADER_BYTES} record bytes, "
                              f"expected {n * dt.itemsize}")
    rec = np.frombuffer(buf, dtype=dt, count=n, offset=HEADER_BYTES)
    head = {"version": version, "flags": flags, "vars": vars_, "edge": edge, "time": time,
            "step": step, "records": n}
    return (head, rec["key"].astype(np.uint64),
            rec["payload"].astype(np.float64).reshape(n, vars_, cells))


def merge(order, parts):
    """Records of several ranks [(keys, payload), ...] into the canonical order
    `order` (Forest.leaves()); every key must appear exactly once."""
    order = np.asarray(order, dtype=np.uint64)
    pos = {int(k): i for i, k in enumerate(order)}
    first = next(p for _, p in parts if len(p))
    out = np.empty((len(order),) + np.asarray(first).shape[1:], dtype=np.float64)
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


def save(path, forest, time: float = 0.0, step: int = 0, state=None, keys=None,
         group=None) -> bytes | None:
    """Write the forest's interior state (device arena, or `state` [local][V][E^3]
    if given, for the leaves `keys`, default this rank's leaves). Collective when
    torch.distributed is initialised with more than one rank: every rank's
    records are gathered and rank 0 writes them in canonical order. Returns the
    bytes on the writing rank, None elsewhere."""
    import torch.distributed as tdist

    local = forest.get_interior() if state is None else np.asarray(state, dtype=np.float64)
    if tdist.is_available() and tdist.is_initialized() and tdist.get_world_size(group) > 1:
        keys = forest.local_leaves() if keys is None else keys
        parts = [None] * tdist.get_world_size(group)
        tdist.all_gather_object(parts, (keys, local), group=group)
        if tdist.get_rank(group) != 0:
            return None
        keys, local = merge(forest.leaves(), parts)
    elif keys is None:
        keys = forest.local_leaves()
    buf = encode(keys, local, time, step)
    if path is not None:
        with open(path, "wb") as fh:
            fh.write(buf)
    return buf


def load(path, forest, stream=None):
    """Read a checkpoint into the forest's device arena (this rank's leaves):
    the records must cover the forest's leaves exactly. Returns the header."""
    with open(path, "rb") as fh:
        head, keys, payload = decode(fh.read())
    if head["vars"] != forest.vars or head["edge"] != forest.edge:
        raise CheckpointError(f"checkpoint is V={head['vars']} E={head['edge']}, forest "
                              f"V={forest.vars} E={forest.edge}")
    _, full = merge(forest.leaves(), [(keys, payload)])
    pos = {int(k): i for i, k in enumerate(forest.leaves())}
    local = full[[pos[int(k)] for k in forest.local_leaves()]]
    forest.set_interior(np.ascontiguousarray(local), stream=stream)
    return head
