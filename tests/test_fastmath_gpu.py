"""Branch-free FP64 division / sqrt (csrc/fastmath.cuh) == IEEE `/` and
`sqrt` bitwise on every operand inside the fast path's range, over billions of
random operands; outside the range the kernel falls back to the IEEE ops."""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode,n", [(0, 1 << 31), (1, 1 << 31), (2, 1 << 30), (3, 1 << 31),
                                    (4, 1 << 31)])
def test_fastmath_bitwise(mode, n):
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "tools", "probes"))
    import probe  # tools/probes/libtmprobe.so: the self-test is not in the product library

    f = probe.load().tmgpu_selftest_fastmath
    bad, chk = C.c_ulonglong(0), C.c_ulonglong(0)
    first = (C.c_double * 2)()
    assert f(mode, n, 0x2412_15518 + mode, C.byref(bad), C.byref(chk), first, None) == 0
    assert chk.value > n // 4
    assert bad.value == 0, (bad.value, chk.value, first[0], first[1])
