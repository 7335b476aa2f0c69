"""ctypes access to tools/probes/libtmprobe.so (diagnostics, not the product):
the FP64 DFMA / DMMA peak microbenchmarks and the fastmath.cuh self-test."""
import ctypes as C
import os

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtmprobe.so")


def load():
    if not os.path.exists(PATH):
        raise FileNotFoundError(f"{PATH} not built (make -C tools/probes)")
    lib = C.CDLL(PATH)
    lib.tmgpu_fp64_peak.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p]
    lib.tmgpu_fp64_probe.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
    lib.tmgpu_dmma_probe.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
    lib.tmgpu_dfma3_probe.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_double)]
    lib.tmgpu_selftest_fastmath.restype = C.c_int
    lib.tmgpu_selftest_fastmath.argtypes = [C.c_int, C.c_longlong, C.c_uint64, C.POINTER(C.c_ulonglong),
                                            C.POINTER(C.c_ulonglong), C.POINTER(C.c_double), C.c_void_p]
    return lib


def fp64_peaks():
    """(DFMA TFLOP/s: 8 warps x 8 chains per SM-slot kernel, DMMA m8n8k4 TFLOP/s at
    16 warps x 8 accumulators per SM) measured now on the current device."""
    lib = load()
    tf, ms = C.c_double(0), C.c_double(0)
    if lib.tmgpu_fp64_peak(20000, C.byref(tf), C.byref(ms), None) != 0:
        raise RuntimeError("DFMA peak probe failed")
    dm = C.c_double(0)
    if lib.tmgpu_dmma_probe(16, 8, 20000, C.byref(dm)) != 0:
        raise RuntimeError("DMMA peak probe failed")
    return tf.value, dm.value
