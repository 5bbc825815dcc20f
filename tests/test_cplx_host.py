"""The device complex ops (csrc/cplx.cuh), compiled for the host, against glibc /
CPython semantics.  m_hypot is a port of glibc's __hypot; it must agree with
libm bit for bit, or the device pivot search would diverge from the reference."""

import cmath
import ctypes
import math
import os
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def shim(tmp_path_factory):
    out = tmp_path_factory.mktemp("shim") / "libshim.so"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", str(out),
                    os.path.join(HERE, "cplx_host_shim.cpp")], check=True)
    lib = ctypes.CDLL(str(out))
    lib.shim_hypot.restype = ctypes.c_double
    lib.shim_hypot.argtypes = [ctypes.c_double, ctypes.c_double]
    dp = ctypes.POINTER(ctypes.c_double)
    lib.shim_div.argtypes = [dp, dp, dp]
    lib.shim_sqrt.argtypes = [dp, dp]
    lib.shim_rdiv.argtypes = [dp, ctypes.c_double, dp, dp]
    return lib


def test_hypot_bit_exact_vs_libm(shim):
    libm = ctypes.CDLL("libm.so.6")
    libm.hypot.restype = ctypes.c_double
    libm.hypot.argtypes = [ctypes.c_double, ctypes.c_double]
    rng = np.random.default_rng(7)
    n = 200_000
    x = rng.normal(size=n) * 2.0 ** rng.integers(-40, 40, n)
    y = np.where(rng.random(n) < 0.5, x * rng.uniform(0.3, 3, n),
                 rng.normal(size=n) * 2.0 ** rng.integers(-40, 40, n))
    # scaling branches and special values
    ext = rng.normal(size=4000) * 2.0 ** rng.integers(-1070, 1020, 4000)
    x = np.concatenate([x, ext, [0.0, -0.0, 1.0, np.inf, -np.inf, np.nan, 3.0, 1e-320]])
    y = np.concatenate([y, ext[::-1], [0.0, 1.0, 0.0, 1.0, np.nan, 2.0, 4.0, 1e-310]])
    bad = 0
    for a, b in zip(x, y):
        r1, r2 = shim.shim_hypot(a, b), libm.hypot(a, b)
        if not (r1 == r2 or (math.isnan(r1) and math.isnan(r2))):
            bad += 1
    assert bad == 0


def _c(z):
    return (ctypes.c_double * 2)(z.real, z.imag)


def test_div_is_cpython_quot(shim):
    """CPython's complex division is _Py_c_quot, the same algorithm numba uses."""
    rng = np.random.default_rng(8)
    out = (ctypes.c_double * 2)()
    for _ in range(20000):
        a = complex(*rng.normal(size=2) * 10.0 ** rng.integers(-5, 5, 2))
        b = complex(*rng.normal(size=2) * 10.0 ** rng.integers(-5, 5, 2))
        shim.shim_div(_c(a), _c(b), out)
        q = a / b
        assert (out[0], out[1]) == (q.real, q.imag)


def test_sqrt_matches_numpy_csqrt_for_finite(shim):
    rng = np.random.default_rng(9)
    out = (ctypes.c_double * 2)()
    worst = 0.0
    for _ in range(5000):
        z = complex(*rng.normal(size=2))
        shim.shim_sqrt(_c(z), out)
        r = complex(out[0], out[1])
        worst = max(worst, abs(r - cmath.sqrt(z)) / abs(cmath.sqrt(z)))
    assert worst < 4e-16


def test_rdiv_is_div_by_real_bit_for_bit(shim):
    """m_rdiv (complex / real, the ratio and denominator folded) returns exactly the bits
    of the general Smith division by (r, 0), special values and signed zeros included."""
    rng = np.random.default_rng(10)
    vals = [0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, np.nan, 5e-324, -5e-324, 1e308, -1e-308]
    A = [complex(a, b) for a in vals for b in vals]
    A += [complex(*rng.normal(size=2) * 10.0 ** rng.integers(-300, 300, 2)) for _ in range(20000)]
    R = vals + list(rng.normal(size=2000) * 10.0 ** rng.integers(-300, 300, 2000))
    out, ref = (ctypes.c_double * 2)(), (ctypes.c_double * 2)()
    bad = 0
    for i, a in enumerate(A):
        for r in (R[i % len(R)], R[(7 * i + 3) % len(R)]):
            shim.shim_rdiv(_c(a), r, out, ref)
            got = np.array([out[0], out[1]]).view(np.uint64)
            exp = np.array([ref[0], ref[1]]).view(np.uint64)
            same = (got == exp) | (np.isnan([out[0], out[1]]) & np.isnan([ref[0], ref[1]]))
            bad += int(not same.all())
    assert bad == 0
