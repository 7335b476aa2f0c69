"""Hydro stage API — a drop-in mirror of the reference ``taskmesh::hydro``
interface (proj/include/taskmesh/hydro/stage.hpp, rk3.hpp), backed by the
sm_100a kernels in libtmgpu.so.

Same names, argument meaning and error behaviour as the reference:
``StageGeom``/``StageParams``/``Mode``, ``encode_header``/``decode_header``
(stage.cpp:10-29), ``stage_subgrid`` (stage.hpp:68-71), ``make_stage_kernel``
returning a fusable ``KernelSpec`` (stage.hpp:73-75, aggregator.hpp:94-106),
``max_wavespeed`` (stage.hpp:77-80), ``rk3_combine`` + ``kStageFluxWeight``
(rk3.hpp:16-34), and ``SolverError`` raised with the reference's message on a
non-finite state (stage.cpp:209-216).

Buffers may be numpy arrays (host memory: the call stages through device
memory, H2D + kernel + D2H) or CUDA torch tensors (device memory: the launch
runs on the current torch stream). float64, C-contiguous.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np

from . import _lib
from ._lib import TmgpuError, lib

kHeaderDoubles = 8
kRhoFloor = 1e-10
kPressureFloor = 1e-12
kDefaultGamma = 7.0 / 5.0
kStageFluxWeight = (1.0, 0.25, 2.0 / 3.0)


class SolverError(RuntimeError):
    """Non-finite state after a stage (reference hydro::SolverError)."""


class Mode(enum.IntEnum):
    scalar = 0
    euler = 1


@dataclass
class StageParams:
    mode: Mode = Mode.scalar
    dx: float = 1.0
    dt: float = 0.0
    gamma: float = kDefaultGamma
    advect: Sequence[float] = field(default_factory=lambda: (1.0, 0.0, 0.0))


@dataclass(frozen=True)
class StageGeom:
    edge: int = 8
    ghost: int = 2
    vars: int = 1

    def stride(self) -> int:
        return self.edge + 2 * self.ghost

    def ghosted_elems(self) -> int:
        return self.vars * self.stride() ** 3

    def in_slice(self) -> int:
        return kHeaderDoubles + self.ghosted_elems()

    def interior_elems(self) -> int:
        return self.vars * self.edge ** 3

    def face_elems(self) -> int:
        return self.vars * self.edge ** 2

    def face_offset(self, axis: int, side: int) -> int:
        return self.interior_elems() + (2 * axis + side) * self.face_elems()

    def diag_offset(self) -> int:
        return self.interior_elems() + 6 * self.face_elems()

    def out_slice(self) -> int:
        return self.diag_offset() + 1


def encode_header(p: StageParams, out) -> None:
    """stage.cpp:10-19."""
    out[0] = float(int(p.mode))
    out[1] = p.dx
    out[2] = p.dt
    out[3] = p.gamma
    out[4], out[5], out[6] = (float(a) for a in p.advect)
    out[7] = 0.0


def decode_header(h) -> StageParams:
    """stage.cpp:21-29."""
    h = [float(x) for x in h[:kHeaderDoubles]]
    return StageParams(Mode.scalar if h[0] == 0.0 else Mode.euler, h[1], h[2], h[3],
                       (h[4], h[5], h[6]))


# ------------------------------------------------------------------ buffers
def _addr(x):
    """(pointer, host?, stream, numel) for a numpy array or torch tensor."""
    if isinstance(x, np.ndarray):
        if x.dtype != np.float64 or not x.flags["C_CONTIGUOUS"]:
            raise ValueError("buffers must be C-contiguous float64")
        return x.ctypes.data, True, None, x.size
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(x, torch.Tensor):
        if x.dtype != torch.float64 or not x.is_contiguous():
            raise ValueError("buffers must be contiguous float64")
        if x.is_cuda:
            return x.data_ptr(), False, torch.cuda.current_stream(x.device).cuda_stream, x.numel()
        return x.data_ptr(), True, None, x.numel()
    raise TypeError(f"unsupported buffer type {type(x)!r}")


def _flags(host: bool, fast: bool) -> int:
    return (_lib.TMGPU_HOST_PTRS if host else 0) | (_lib.TMGPU_FAST if fast else 0)


def stage_fused(packed_in, packed_out, in_slice: int, out_slice: int, count: int,
                geom: StageGeom, fast: bool = False) -> None:
    """One aggregated launch over `count` packed [header|state] slices."""
    pi, hi, st, ni = _addr(packed_in)
    po, ho, _, no = _addr(packed_out)
    if hi != ho:
        raise ValueError("input and output must both be host or both be device buffers")
    if ni < count * in_slice or no < count * out_slice:
        raise ValueError("buffer smaller than count slices")
    err = TmgpuError()
    rc = lib.tmgpu_stage_fused(pi, po, in_slice, out_slice, count, geom.edge, geom.ghost,
                               geom.vars, _flags(hi, fast), st, C.byref(err))
    _lib.check(rc, err, SolverError)


def stage_subgrid(p: StageParams, geom: StageGeom, lane_width: int, in_ghosted, out,
                  fast: bool = False) -> None:
    """stage.hpp:68-71: one stage on one sub-grid (lane_width is ignored)."""
    if lane_width not in (1, 2, 4, 8, 16):
        raise ValueError("lane width must be 1, 2, 4, 8 or 16")  # lanes.hpp:212-213
    h = np.zeros(kHeaderDoubles)
    encode_header(p, h)
    pi, hi, st, _ = _addr(in_ghosted)
    po, ho, _, _ = _addr(out)
    if hi != ho:
        raise ValueError("input and output must both be host or both be device buffers")
    err = TmgpuError()
    if hi:
        rc = lib.tmgpu_stage_subgrid(h.ctypes.data, geom.edge, geom.ghost, geom.vars, lane_width,
                                     pi, po, _flags(True, fast), None, C.byref(err))
    else:
        rc = lib.tmgpu_stage_subgrid(h.ctypes.data, geom.edge, geom.ghost, geom.vars, lane_width,
                                     pi, po, _flags(False, fast), st, C.byref(err))
    _lib.check(rc, err, SolverError)


KernelFn = Callable[[object, object, int, int, int], None]


@dataclass
class KernelSpec:
    """aggregator.hpp:101-106."""
    id: int = 0
    in_slice: int = 0
    out_slice: int = 0
    fn: KernelFn | None = None


def make_stage_kernel(geom: StageGeom, lane_width: int, kernel_id: int,
                      fast: bool = False) -> KernelSpec:
    """stage.cpp:229-246: the stage as a fusable kernel whose fn runs one
    aggregated sm_100a launch over all slices of the batch."""
    if lane_width not in (1, 2, 4, 8, 16):
        raise ValueError("lane width must be 1, 2, 4, 8 or 16")

    def fn(packed_in, packed_out, in_slice, out_slice, count):
        stage_fused(packed_in, packed_out, in_slice, out_slice, count, geom, fast)

    return KernelSpec(kernel_id, geom.in_slice(), geom.out_slice(), fn)


def max_wavespeed(p: StageParams, geom: StageGeom, ghosted) -> float:
    """stage.cpp:248-272."""
    if p.mode == Mode.scalar:
        a = [float(x) for x in p.advect]
        return float(np.sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]))
    g = np.ascontiguousarray(np.asarray(ghosted, dtype=np.float64))
    slice_ = np.empty(geom.in_slice())
    encode_header(p, slice_)
    slice_[kHeaderDoubles:] = g.reshape(-1)[: geom.ghosted_elems()]
    res = np.zeros(1)
    err = TmgpuError()
    rc = lib.tmgpu_max_wavespeed(slice_.ctypes.data, geom.in_slice(), 1, geom.edge, geom.ghost,
                                 geom.vars, res.ctypes.data, _lib.TMGPU_HOST_PTRS, None,
                                 C.byref(err))
    _lib.check(rc, err)
    return float(res[0])


def rk3_combine(stage: int, u0, v):
    """rk3.hpp:18-27, elementwise on the device (scalars or arrays)."""
    scalar = np.isscalar(u0) and np.isscalar(v)
    a = np.ascontiguousarray(np.atleast_1d(np.asarray(u0, dtype=np.float64)))
    b = np.ascontiguousarray(np.atleast_1d(np.asarray(v, dtype=np.float64)))
    out = np.empty_like(b)
    err = TmgpuError()
    rc = lib.tmgpu_rk3_combine(stage, a.ctypes.data, b.ctypes.data, out.ctypes.data, out.size,
                               _lib.TMGPU_HOST_PTRS, None, C.byref(err))
    _lib.check(rc, err)
    return float(out[0]) if scalar else out
