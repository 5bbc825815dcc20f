"""ctypes wrapper around referee.c -- TEST INFRASTRUCTURE ONLY.

The extended-precision referee that adjudicates between double-precision
evaluations of the hafnian subset sum (the reference, MIRROR, FAST).  Used by
tests/golden/gen_referee.py (fixture generation, run in the build container)
and by tests/; never by the product package.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_libs = {}

_dp = ctypes.POINTER(ctypes.c_double)
_u64p = ctypes.POINTER(ctypes.c_uint64)


def lib(quad: bool = False):
    name = "libreferee_q.so" if quad else "libreferee.so"
    if name not in _libs:
        path = os.path.join(_HERE, name)
        src = os.path.join(_HERE, "referee.c")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
            subprocess.run(["make", "-s", "-C", _HERE, name], check=True)
        L = ctypes.CDLL(path)
        L.ref_sum_range.argtypes = [_dp, _dp, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                    ctypes.c_int, ctypes.c_int, _dp]
        L.ref_sum_range.restype = ctypes.c_int
        L.ref_terms.argtypes = [_dp, _dp, ctypes.c_int, _u64p, ctypes.c_int64, ctypes.c_int,
                                ctypes.c_int, _dp]
        L.ref_terms.restype = ctypes.c_int
        L.ref_mant_bits.restype = ctypes.c_int
        _libs[name] = L
    return _libs[name]


def _threads(threads):
    return threads or len(os.sched_getaffinity(0))


def sum_range(atilde, diag, n_half, lo, hi, include_loops, threads=None, quad=False):
    """Referee sum of the signed terms of masks [lo, hi) (mask 0 skipped).

    Returns (value_hi, value_lo, abs_sum): value_hi + value_lo (complex128 each)
    represents the extended-precision sum; abs_sum = sum |t|."""
    at = np.ascontiguousarray(atilde, np.complex128)
    dg = np.ascontiguousarray(diag, np.complex128)
    out = np.zeros(5)
    rc = lib(quad).ref_sum_range(at.ctypes.data_as(_dp), dg.ctypes.data_as(_dp), int(n_half),
                                 int(lo), int(hi), int(bool(include_loops)), _threads(threads),
                                 out.ctypes.data_as(_dp))
    if rc != 0:
        raise ValueError("referee rejected the arguments")
    return complex(out[0], out[2]), complex(out[1], out[3]), float(out[4])


def terms(atilde, diag, n_half, masks, include_loops, threads=None, quad=False):
    """Referee values (rounded to complex128) of the terms of `masks`."""
    at = np.ascontiguousarray(atilde, np.complex128)
    dg = np.ascontiguousarray(diag, np.complex128)
    mk = np.ascontiguousarray(masks, np.uint64)
    out = np.zeros(mk.size, np.complex128)
    rc = lib(quad).ref_terms(at.ctypes.data_as(_dp), dg.ctypes.data_as(_dp), int(n_half),
                             mk.ctypes.data_as(_u64p), mk.size, int(bool(include_loops)),
                             _threads(threads), out.ctypes.data_as(_dp))
    if rc != 0:
        raise ValueError("referee rejected the arguments")
    return out


def rel_err(value, hi, lo=0j) -> float:
    """|value - (hi + lo)| / |hi + lo|, with the difference taken against hi first
    (exact for value near hi) so the referee's extra digits are not lost."""
    d = (complex(value) - hi) - lo
    return abs(d) / abs(hi)
