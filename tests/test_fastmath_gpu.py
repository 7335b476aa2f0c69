"""Branch-free FP64 division / sqrt (csrc/fastmath.cuh) == IEEE `/` and
`sqrt` bitwise on every operand inside the fast path's range, over billions of
random operands; outside the range the kernel falls back to the IEEE ops."""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode,n", [(0, 1 << 31), (1, 1 << 31), (2, 1 << 30), (3, 1 << 31),
                                    (4, 1 << 31)])
def test_fastmath_bitwise(mode, n):
    from paper_2412_15518_b200 import _lib

    f = _lib.lib.tmgpu_selftest_fastmath
    f.restype = C.c_int
    f.argtypes = [C.c_int, C.c_longlong, C.c_uint64, C.POINTER(C.c_ulonglong),
                  C.POINTER(C.c_ulonglong), C.POINTER(C.c_double), C.c_void_p]
    bad, chk = C.c_ulonglong(0), C.c_ulonglong(0)
    first = (C.c_double * 2)()
    assert f(mode, n, 0x2412_15518 + mode, C.byref(bad), C.byref(chk), first, None) == 0
    assert chk.value > n // 4
    assert bad.value == 0, (bad.value, chk.value, first[0], first[1])
