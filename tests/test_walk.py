"""fl_walk (csrc/walk.h) == k sequential IEEE additions, the reference's
row-incremental coordinate walk (image_ops.cpp:124-131)."""
import ctypes
import os

import pytest

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build", "libwalktest.so")


@pytest.mark.skipif(not os.path.exists(LIB), reason="build/libwalktest.so not built (make)")
@pytest.mark.parametrize("smax", [1.0, 40.0, 2500.0, 30000.0])
def test_walk_matches_brute_force(smax):
    lib = ctypes.CDLL(LIB)
    lib.walk_check.restype = ctypes.c_longlong
    lib.walk_check.argtypes = [ctypes.c_uint64, ctypes.c_longlong, ctypes.c_int, ctypes.c_double,
                               ctypes.POINTER(ctypes.c_double)]
    worst = ctypes.c_double(0)
    assert lib.walk_check(17, 4000, 4100, smax, ctypes.byref(worst)) == 0, worst.value
