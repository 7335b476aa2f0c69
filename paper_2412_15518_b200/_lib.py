"""ctypes binding of libtmgpu.so (the C ABI declared in include/tmgpu.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no CPU fallback: importing the package without the built library
raises, and every compute call on a machine without a usable B200 returns
TMGPU_ERR_CUDA, surfaced here as ``CudaError``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtmgpu.so")

TMGPU_OK = 0
TMGPU_ERR_SOLVER = 1
TMGPU_ERR_INVALID = 2
TMGPU_ERR_CUDA = 3
TMGPU_ERR_AMR = 4
TMGPU_ERR_AGG = 5

TMGPU_HOST_PTRS = 0x1
TMGPU_FAST = 0x2
TMGPU_ASYNC = 0x4
TMGPU_EXACT_GHOSTS = 0x8
TMGPU_GRAV_AM = 0x100
TMGPU_OVERLAP = 0x10
TMGPU_NO_GRAPH = 0x20


class TmgpuError(C.Structure):
    _fields_ = [("code", C.c_int), ("cell", C.c_int * 3), ("slice", C.c_int64),
                ("message", C.c_char * 256)]


class CudaError(RuntimeError):
    """A CUDA runtime failure inside libtmgpu (no GPU, launch error, ...)."""


if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback for the B200 kernels)")

lib = C.CDLL(LIB_PATH)

_dp = C.POINTER(C.c_double)
_vp = C.c_void_p
_ep = C.POINTER(TmgpuError)


def _sig(name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args
    return f


_sig("tmgpu_in_slice", C.c_size_t, [C.c_int] * 3)
_sig("tmgpu_out_slice", C.c_size_t, [C.c_int] * 3)
_sig("tmgpu_stage_fused", C.c_int, [_vp, _vp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_int,
                                    C.c_int, C.c_int, C.c_int, _vp, _ep])
_sig("tmgpu_stage_subgrid", C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_uint, _vp, _vp,
                                      C.c_int, _vp, _ep])
_sig("tmgpu_max_wavespeed", C.c_int, [_vp, C.c_size_t, C.c_size_t, C.c_int, C.c_int, C.c_int,
                                      _vp, C.c_int, _vp, _ep])
_sig("tmgpu_rk3_combine", C.c_int, [C.c_int, _vp, _vp, _vp, C.c_size_t, C.c_int, _vp, _ep])
_sig("tmgpu_version", C.c_char_p, [])
_sig("tmgpu_launch_count", C.c_uint64, [])


def launch_count() -> int:
    return int(lib.tmgpu_launch_count())


def check(rc: int, err: TmgpuError, solver_exc=RuntimeError):
    """Map a C-ABI return code to the reference's exception types."""
    if rc == TMGPU_OK:
        return
    msg = err.message.decode(errors="replace")
    if rc == TMGPU_ERR_SOLVER:
        raise solver_exc(msg)
    if rc == TMGPU_ERR_CUDA:
        raise CudaError(msg)
    if rc == TMGPU_ERR_INVALID:
        raise ValueError(msg)
    raise RuntimeError(f"tmgpu error {rc}: {msg}")
