"""Device ports of glibc exp/log/sincos and of the reference RNG, compared bit
for bit with the host glibc (the reference's libm) and with the reference's
own rng.cpp (oracle/_ref)."""
import ctypes as C
import os

import numpy as np
import pytest

import ref
from paper_2411_16445_b200 import _abi as A

pytestmark = pytest.mark.gpu

_G = None


def glibc(func, x):
    global _G
    if _G is None:
        _G = C.CDLL(os.path.join(os.path.dirname(ref.__file__), "_ref", "libglibc_eval.so"))
    x = np.ascontiguousarray(x, np.float64)
    out = np.empty_like(x)
    _G.glibc_eval(C.c_int(func), x.ctypes.data_as(C.c_void_p), C.c_int64(len(x)),
                  out.ctypes.data_as(C.c_void_p))
    return out


def device(func, x=None, key=(0, 0, 0, 0), n0=0, n=None):
    n = len(x) if x is not None else n
    out = np.empty(n, np.float64)
    k = (C.c_uint64 * 4)(*key)
    xi = None if x is None else np.ascontiguousarray(x, np.float64)
    st = A.lib().mcg_device_math(0, func, None if xi is None else xi.ctypes.data_as(C.c_void_p),
                                 n, k, n0, out.ctypes.data_as(C.c_void_p))
    assert st == 0, A.lib().mcg_last_error()
    return out


def bits_equal(a, b):
    return np.array_equal(a.view(np.uint64), b.view(np.uint64))


RNG = np.random.default_rng(12345)
N = 4_000_000


@pytest.mark.parametrize("lo,hi", [(-20, 20), (-1, 1), (-745.2, -700), (700, 709.7), (-1e-3, 1e-3)])
def test_exp_matches_glibc(gpu, lo, hi):
    x = RNG.uniform(lo, hi, N)
    assert bits_equal(device(0, x), glibc(0, x))


def test_log_matches_glibc(gpu):
    u1 = ((RNG.integers(0, 2**53, N, dtype=np.uint64)).astype(np.float64) + 1.0) * 2.0**-53
    assert bits_equal(device(1, u1), glibc(1, u1))
    x = RNG.uniform(0.9, 1.1, N)
    assert bits_equal(device(1, x), glibc(1, x))


@pytest.mark.parametrize("lo,hi", [(0, 6.283185307179586), (-0.9, 0.9), (0.8, 2.5), (2.4, 7)])
def test_sincos_matches_glibc(gpu, lo, hi):
    x = RNG.uniform(lo, hi, N)
    assert bits_equal(device(2, x), glibc(2, x))
    assert bits_equal(device(3, x), glibc(3, x))


@pytest.mark.parametrize("key", [(9, 9, 9, 9), (1, 2, 3, 4), (11, 37, (2 << 32) | 0, 5)])
def test_rng_matches_reference(gpu, key):
    n = 20000
    du = device(4, key=key, n=n)
    dn = device(5, key=key, n=n)
    ru = np.array([ref.uniform_for(key, i) for i in range(n)])
    rn = np.array([ref.normal_for(key, i) for i in range(n)])
    assert bits_equal(du, ru)
    assert bits_equal(dn, rn)
