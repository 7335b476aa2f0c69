"""paper_2412_15518_b200 — B200-native (sm_100a, FP64) per-subgrid hot path of
the AMR hydro mini-app of arXiv 2412.15518 (reference: "taskmesh").

Drop-in for the reference's subgrid-kernel API (see include/tmgpu.h and
INTEGRATION.md). Import fails loudly when libtmgpu.so is not built.
"""
from . import _lib  # noqa: F401  (raises ImportError when the library is missing)
from . import hydro  # noqa: F401

__all__ = ["hydro"]
