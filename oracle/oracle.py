"""ctypes wrapper around the C oracle (hafnian_oracle.c).  TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module; the product package never does.  Every function mirrors one
function of the reference kernel module (pkg/src/hafnium/kernels/_numba.py)
and returns numpy complex128 data in the same layout.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u64p = ctypes.POINTER(ctypes.c_uint64)


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "hafnian_oracle.c"))
    ):
        subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        c_int, c_u64, c_i64 = ctypes.c_int, ctypes.c_uint64, ctypes.c_int64
        L.orc_subset_term.argtypes = [_dp, _dp, c_int, c_u64, c_int, c_int, c_int, _dp]
        L.orc_subset_term.restype = c_int
        L.orc_terms.argtypes = [_dp, _dp, c_int, _u64p, c_i64, c_int, c_int, c_int, c_int, _dp, _i32p]
        L.orc_terms.restype = None
        L.orc_sum_subsets_det.argtypes = [_dp, _dp, c_int, c_int, c_int, c_int, c_int, c_int, _dp, _i64p]
        L.orc_sum_subsets_fast.argtypes = L.orc_sum_subsets_det.argtypes
        L.orc_sum_mask_range.argtypes = [_dp, _dp, c_int, c_u64, c_u64, c_int, c_int, c_int, c_int,
                                         c_int, _dp, _i64p]
        L.orc_tree_reduce.argtypes = [_dp, c_i64, _dp]
        L.orc_power_traces_charpoly.argtypes = [_dp, c_int, c_int, _dp]
        L.orc_power_traces_charpoly.restype = c_int
        L.orc_charpoly_coefficients.argtypes = [_dp, c_int, _dp]
        L.orc_power_traces_spectral.argtypes = [_dp, c_int, c_int, c_int, _dp, _i64p]
        L.orc_power_traces_spectral.restype = c_int
        L.orc_exp_top.argtypes = [_dp, c_int, _dp]
        L.orc_hypot.argtypes = [ctypes.c_double, ctypes.c_double]
        L.orc_hypot.restype = ctypes.c_double
        _lib = L
    return _lib


def _c(a, dtype=np.complex128):
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a, t=_dp):
    return a.ctypes.data_as(t)


def subset_term(atilde, diag, mask, n_half, backend, include_loops, cap_mult=30):
    at, dg = _c(atilde), _c(diag)
    out = np.zeros(1, np.complex128)
    st = lib().orc_subset_term(_p(at), _p(dg), n_half, int(mask), backend, int(include_loops),
                               cap_mult, _p(out))
    return complex(out[0]), int(st)


def terms(atilde, diag, n_half, masks, backend=1, include_loops=False, cap_mult=30, threads=None):
    at, dg = _c(atilde), _c(diag)
    mk = _c(masks, np.uint64)
    out = np.zeros(mk.size, np.complex128)
    st = np.zeros(mk.size, np.int32)
    lib().orc_terms(_p(at), _p(dg), n_half, _p(mk, _u64p), mk.size, backend, int(include_loops),
                    cap_mult, threads or os.cpu_count(), _p(out), _p(st, _i32p))
    return out, st


def sum_subsets_det(atilde, diag, n_half, backend, include_loops, workers, n_ranges, cap_mult=30):
    at, dg = _c(atilde), _c(diag)
    sums = np.zeros(n_ranges, np.complex128)
    fails = np.zeros(n_ranges, np.int64)
    lib().orc_sum_subsets_det(_p(at), _p(dg), n_half, backend, int(include_loops), workers,
                              n_ranges, cap_mult, _p(sums), _p(fails, _i64p))
    return sums, fails


def sum_subsets_fast(atilde, diag, n_half, backend, include_loops, workers, n_ranges, cap_mult=30):
    at, dg = _c(atilde), _c(diag)
    sums = np.zeros(workers, np.complex128)
    fails = np.zeros(workers, np.int64)
    lib().orc_sum_subsets_fast(_p(at), _p(dg), n_half, backend, int(include_loops), workers,
                               n_ranges, cap_mult, _p(sums), _p(fails, _i64p))
    return sums, fails


def sum_mask_range(atilde, diag, n_half, lo, hi, n_chunks, backend=1, include_loops=False,
                   cap_mult=30, threads=None):
    at, dg = _c(atilde), _c(diag)
    sums = np.zeros(n_chunks, np.complex128)
    fails = np.zeros(n_chunks, np.int64)
    lib().orc_sum_mask_range(_p(at), _p(dg), n_half, lo, hi, n_chunks, backend,
                             int(include_loops), cap_mult, threads or os.cpu_count(), _p(sums),
                             _p(fails, _i64p))
    return sums, fails


def tree_reduce(values) -> complex:
    v = _c(values)
    out = np.zeros(1, np.complex128)
    lib().orc_tree_reduce(_p(v), v.size, _p(out))
    return complex(out[0])


def power_traces_charpoly(b, K):
    h = np.array(b, dtype=np.complex128, order="C")
    out = np.zeros(K, np.complex128)
    ok = lib().orc_power_traces_charpoly(_p(h), h.shape[0], K, _p(out))
    return out, bool(ok)


def charpoly_coefficients(b):
    h = np.array(b, dtype=np.complex128, order="C")
    out = np.zeros(h.shape[0] + 1, np.complex128)
    lib().orc_charpoly_coefficients(_p(h), h.shape[0], _p(out))
    return out


def power_traces_spectral(b, K, cap_mult=30):
    h = np.array(b, dtype=np.complex128, order="C")
    out = np.zeros(K, np.complex128)
    sweeps = np.zeros(1, np.int64)
    conv = lib().orc_power_traces_spectral(_p(h), h.shape[0], K, cap_mult, _p(out),
                                           _p(sweeps, _i64p))
    return out, int(sweeps[0]), bool(conv)


def exp_top(s) -> complex:
    sv = _c(s)
    out = np.zeros(1, np.complex128)
    lib().orc_exp_top(_p(sv), sv.size - 1, _p(out))
    return complex(out[0])


def prepare(A, include_loops):
    """engine._prepare (engine.py:140-150) on an already-symmetric array."""
    a = np.array(A, dtype=np.complex128)
    iu = np.triu_indices(a.shape[0], k=1)
    a[(iu[1], iu[0])] = a[iu]
    if not include_loops:
        np.fill_diagonal(a, 0.0)
    diag = np.ascontiguousarray(np.diag(a))
    n = a.shape[0]
    perm = np.arange(n)
    perm[0::2] += 1
    perm[1::2] -= 1
    return np.ascontiguousarray(a[perm]), diag, n // 2


def hafnian(A, backend=1, include_loops=False, threads=None, n_ranges=512):
    """Full reference pipeline: prepare, sum_subsets_det, tree_reduce."""
    at, dg, nh = prepare(A, include_loops)
    if nh == 0:
        return 1.0 + 0.0j
    nr = min((1 << nh) - 1, n_ranges)
    sums, fails = sum_subsets_det(at, dg, nh, backend, include_loops, threads or os.cpu_count(), nr)
    return tree_reduce(sums), int(fails.max())
