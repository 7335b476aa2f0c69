"""DFMA throughput vs warps per SM and independent chains per thread (the FP64
latency/occupancy trade-off behind the M2L kernel's 8 warps per SM), and the
FP64 tensor-core (DMMA) throughput for comparison."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "probes"))
import probe  # noqa: E402  tools/probes/libtmprobe.so

plib = probe.load()
f = plib.tmgpu_fp64_probe
f.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
for warps in (4, 8, 16, 32):
    row = []
    for chains in (1, 2, 4, 8, 16):
        t = C.c_double()
        f(warps, chains, 20000, C.byref(t))
        row.append(f"{t.value:6.2f}")
    print(f"warps/SM {warps:2d}: chains 1,2,4,8,16 -> TFLOP/s", " ".join(row))

g = plib.tmgpu_dmma_probe
g.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
for warps in (4, 8, 16, 32):
    row = []
    for chains in (1, 2, 4, 8):
        t = C.c_double()
        g(warps, chains, 20000, C.byref(t))
        row.append(f"{t.value:6.2f}")
    print(f"DMMA m8n8k4 warps/SM {warps:2d}: chains 1,2,4,8 -> TFLOP/s", " ".join(row))

h = plib.tmgpu_dfma3_probe
h.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_double)]
row = []
for warps in (4, 8, 16, 32):
    t = C.c_double()
    h(warps, 20000, C.byref(t))
    row.append(f"{t.value:6.2f}")
print("DFMA, three fresh register operands, 8 chains; warps/SM 4,8,16,32 -> TFLOP/s", " ".join(row))
