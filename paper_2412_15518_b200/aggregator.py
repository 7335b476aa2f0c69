"""Kernel-aggregation executor — a mirror of the reference ``taskmesh::agg``
interface (proj/include/taskmesh/aggregator.hpp): ``ExecutorPool`` /
``ExecutorLease`` / ``AggregationRegion`` / ``AggCounters`` / ``KernelRegistry``
/ ``AggError``, with CUDA streams as the executors (csrc/aggregator.cpp).

A region launch is one aggregated kernel over the batch on the pinned
executor's stream (H2D of the packed slices, kernel, D2H); ``submit_slice``
returns a future whose ``get()`` waits for the batch and returns the
slice's output view, raising the batch's error for every slice of a failed
batch (aggregator.cpp:164-167).
"""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _lib
from ._lib import TmgpuError, lib
from .hydro import KernelSpec, SolverError, StageGeom

_vp = C.c_void_p
_ep = C.POINTER(TmgpuError)


def _sig(name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args


_sig("tmgpu_execpool_create", _vp, [C.c_size_t, _ep])
_sig("tmgpu_execpool_destroy", None, [_vp])
_sig("tmgpu_execpool_size", C.c_size_t, [_vp])
_sig("tmgpu_execpool_acquire", C.c_size_t, [_vp])
_sig("tmgpu_execpool_pick_index", C.c_size_t, [_vp])
_sig("tmgpu_execpool_acquire_at", C.c_int, [_vp, C.c_size_t, _ep])
_sig("tmgpu_execpool_release", None, [_vp, C.c_size_t])
_sig("tmgpu_execpool_in_flight", C.c_uint64, [_vp, C.c_size_t])
_sig("tmgpu_region_create", _vp, [_vp, C.c_int, C.c_size_t, C.c_size_t, C.c_int, C.c_int, C.c_int,
                                  C.c_int, C.c_size_t, C.c_size_t, C.POINTER(C.c_uint64), _ep])
_sig("tmgpu_region_create_kernel", _vp, [_vp, _vp, _vp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t,
                                         C.POINTER(C.c_uint64), _ep])
_sig("tmgpu_region_submit", C.c_longlong, [_vp, _vp, C.c_size_t, _ep])
_sig("tmgpu_region_flush", C.c_int, [_vp, _ep])
_sig("tmgpu_region_wait", C.c_int, [_vp, C.c_longlong, _ep])
_sig("tmgpu_region_output", C.POINTER(C.c_double), [_vp, C.c_longlong])
_sig("tmgpu_region_submitted", C.c_size_t, [_vp])
_sig("tmgpu_region_destroy", None, [_vp])


class AggError(ValueError):
    """Reference agg::AggError (a std::logic_error)."""


def _agg_check(rc, err, solver_exc=SolverError):
    if rc == _lib.TMGPU_ERR_AGG:
        raise AggError(err.message.decode())
    _lib.check(rc, err, solver_exc)


class ExecutorLease:
    """RAII in-flight slot on one executor (aggregator.hpp:34-52)."""

    def __init__(self, pool: "ExecutorPool", index: int):
        self._pool, self._index = pool, index

    def index(self) -> int:
        return self._index

    def reset(self) -> None:
        if self._pool is not None:
            lib.tmgpu_execpool_release(self._pool.h, self._index)
            self._pool = None

    def __del__(self):
        self.reset()


class ExecutorPool:
    """Pool of CUDA-stream executors with in-flight counters (aggregator.hpp:57-85)."""

    def __init__(self, count: int):
        err = TmgpuError()
        self.h = lib.tmgpu_execpool_create(count, C.byref(err))
        if not self.h:
            raise AggError(err.message.decode())

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:  # lib is None at interpreter exit
            lib.tmgpu_execpool_destroy(self.h)
            self.h = None

    def size(self) -> int:
        return int(lib.tmgpu_execpool_size(self.h))

    def acquire(self) -> ExecutorLease:
        return ExecutorLease(self, int(lib.tmgpu_execpool_acquire(self.h)))

    def pick_index(self) -> int:
        return int(lib.tmgpu_execpool_pick_index(self.h))

    def acquire_at(self, index: int) -> ExecutorLease:
        err = TmgpuError()
        _agg_check(lib.tmgpu_execpool_acquire_at(self.h, index, C.byref(err)), err)
        return ExecutorLease(self, index)

    def in_flight(self, index: int) -> int:
        return int(lib.tmgpu_execpool_in_flight(self.h, index))


class AggCounters:
    """launches / fused_slices / solo_launches (aggregator.hpp:87-92)."""

    def __init__(self):
        self._buf = (C.c_uint64 * 3)()

    @property
    def launches(self) -> int:
        return int(self._buf[0])

    @property
    def fused_slices(self) -> int:
        return int(self._buf[1])

    @property
    def solo_launches(self) -> int:
        return int(self._buf[2])


class KernelRegistry:
    """Per-locality table of fusable kernels keyed by id (aggregator.hpp:108-116)."""

    def __init__(self):
        self._k: dict[int, KernelSpec] = {}

    def add(self, spec: KernelSpec) -> None:
        if spec.id in self._k:
            raise AggError("kernel id registered twice")
        self._k[spec.id] = spec

    def at(self, kid: int) -> KernelSpec:
        if kid not in self._k:
            raise AggError("unknown kernel id")
        return self._k[kid]


class SliceFuture:
    def __init__(self, region: "AggregationRegion", ticket: int):
        self.region, self.ticket = region, ticket

    def get(self) -> np.ndarray:
        """Wait for the slice's batch; the slice's output values (SliceOutput::values)."""
        r = self.region
        err = TmgpuError()
        _agg_check(lib.tmgpu_region_wait(r.h, self.ticket, C.byref(err)), err)
        p = lib.tmgpu_region_output(r.h, self.ticket)
        return np.ctypeslib.as_array(p, shape=(r.out_slice,))


class DeviceKernel:
    """A device kernel registered like a reference KernelSpec (aggregator.hpp:94-106):
    ``fn`` is the address of a C function with the tmgpu_device_kernel signature
    (include/tmgpu.h) that launches one aggregated kernel over packed device
    slices; ``user`` is passed through."""

    def __init__(self, fn: int, in_slice: int, out_slice: int, user: int | None = None):
        if not fn:
            raise AggError("null kernel function")
        self.fn, self.in_slice, self.out_slice, self.user = fn, in_slice, out_slice, user


class AggregationRegion:
    """Work-aggregation region for one device kernel (aggregator.hpp:138-172).

    kernel: a StageGeom (the hydro stage, make_stage_kernel) or a DeviceKernel."""

    def __init__(self, execs: ExecutorPool, kernel, max_slices: int, capacity_slices: int,
                 counters: AggCounters | None = None, fast: bool = False):
        err = TmgpuError()
        cnt = counters._buf if counters is not None else None
        self.execs, self.counters = execs, counters
        if isinstance(kernel, StageGeom):
            g = kernel
            self.in_slice, self.out_slice = g.in_slice(), g.out_slice()
            self.h = lib.tmgpu_region_create(execs.h, 1, self.in_slice, self.out_slice, g.edge, g.ghost,
                                             g.vars, _lib.TMGPU_FAST if fast else 0, max_slices,
                                             capacity_slices, cnt, C.byref(err))
        elif isinstance(kernel, DeviceKernel):
            self.in_slice, self.out_slice = kernel.in_slice, kernel.out_slice
            self.h = lib.tmgpu_region_create_kernel(execs.h, kernel.fn, kernel.user, kernel.in_slice,
                                                    kernel.out_slice, max_slices, capacity_slices, cnt,
                                                    C.byref(err))
        else:
            raise ValueError("kernel must be a StageGeom or a DeviceKernel")
        if not self.h:
            _agg_check(err.code or _lib.TMGPU_ERR_AGG, err)
        self._lock = threading.Lock()

    def submit_slice(self, data) -> SliceFuture:
        a = np.ascontiguousarray(np.asarray(data, dtype=np.float64))
        err = TmgpuError()
        t = lib.tmgpu_region_submit(self.h, a.ctypes.data, a.size, C.byref(err))
        if t < 0:
            _agg_check(err.code, err)
        return SliceFuture(self, int(t))

    def flush(self) -> None:
        err = TmgpuError()
        _agg_check(lib.tmgpu_region_flush(self.h, C.byref(err)), err)

    def submitted(self) -> int:
        return int(lib.tmgpu_region_submitted(self.h))

    def close(self) -> None:
        if getattr(self, "h", None):
            lib.tmgpu_region_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


def when_all(futures):
    """task::when_all analog: every slice output, in order."""
    return [f.get() for f in futures]
