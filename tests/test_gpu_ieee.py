"""The call-free IEEE sequences of advance_p_lean (csrc/push.cu:
sqrt_rn_nocall, rcp_rn_nocall, div_rn_nocall) against the library sqrt.rn /
rcp.rn / div.rn, bit for bit, exhaustively over every float in the ranges the
push guarantees before using them (the particle update's bit-exactness with
the reference rests on this):

* sqrt(1 + |u|^2) with |u|^2 < 2^40: every float in [1, 2^40];
* 1 / gamma and 2 / (1 + |t|^2), gamma, 1 + |t|^2 in [1, 2^20]: every float;
* (q dt / 2m) / gamma for |q dt / 2m| in [2^-100, 2^100]: every gamma in
  [1, 2^20] for a spread of numerators incl. both range ends;
* the mover's (sigma - q) / r: numerators in [2^-24, 2] x every r in
  [2^-25, 2].
"""
import ctypes as C
import struct

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(x):
    return struct.unpack("<I", struct.pack("<f", x))[0]


@pytest.fixture(scope="module")
def check():
    import paper_2102_13133_b200 as pic
    fn = pic.lib().pic_internal_ieee_check
    fn.argtypes = [C.c_int, C.c_float, C.c_uint, C.c_uint, C.POINTER(C.c_ulonglong)]

    def run(mode, a, lo, hi):
        lo_b, hi_b = bits(lo), bits(hi)
        m = C.c_ulonglong(0)
        pic.check(fn(mode, a, lo_b, hi_b - lo_b + 1, C.byref(m)))
        return m.value
    return run


def test_sqrt_exhaustive(check):
    assert check(0, 0.0, 1.0, 2.0 ** 40) == 0


def test_rcp_exhaustive(check):
    assert check(1, 0.0, 1.0, 2.0 ** 20) == 0


@pytest.mark.parametrize("a", [2.0, 2.0 ** -100, -(2.0 ** -100), 2.0 ** 100, -(2.0 ** 100), 0.25 / 2,
                               -0.25 / 2 / 100, 1e-20 * 0.25 / (2 / 64), 3.3e-7, -0.77, 123.456])
def test_div_boris_exhaustive(check, a):
    a = float(np.float32(a))
    assert check(2, a, 1.0, 2.0 ** 20) == 0


@pytest.mark.parametrize("a", [2.0 ** -24, 3 * 2.0 ** -24, 1e-5, 0.1, 0.5, 0.999999, 1.0, 1.5, 1.9999999, 2.0])
def test_div_mover_exhaustive(check, a):
    a = float(np.float32(a))
    assert check(2, a, 2.0 ** -25, 2.0) == 0
    assert check(2, -a, 2.0 ** -25, 2.0) == 0
