"""The reference's kernel-module contract, implemented on the B200.

hafnium.kernels.active() returns a module with this surface
(pkg/src/hafnium/kernels/_numba.py:297-440); this module
provides the same names, argument meanings, return layouts and status
conventions, computed by the sm_100a kernels behind libhafb200.so.  It can be
dropped behind the reference's selector or used through this
package's own engine.

Extra keyword-only arguments (defaults keep the reference call sites valid):
``arith`` ("mirror": the reference's exact IEEE operation sequence, bit-identical
results; "fast": FMA-contracted kernels) and ``device`` (CUDA ordinal).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib

SWEEP_CAP_MULT = 30  # _numba.py:33; read at call time by the engine (monkeypatchable)
DEFLATION_RTOL = 1e-14  # _numba.py:32 (compiled into the kernels)
MAX_HALF = 32  # device masks are 32-bit: n <= 64

ARITH_MODES = {"mirror": 0, "fast": 1}


def default_arith() -> str:
    a = os.environ.get("HAFB200_ARITH", "mirror").strip().lower()
    if a not in ARITH_MODES:
        raise ValueError(f"HAFB200_ARITH must be one of {tuple(ARITH_MODES)}, got {a!r}")
    return a


def _arith_id(arith) -> int:
    a = default_arith() if arith is None else arith
    if a not in ARITH_MODES:
        raise ValueError(f"arith must be one of {tuple(ARITH_MODES)}, got {a!r}")
    return ARITH_MODES[a]


def device_count() -> int:
    """Visible CUDA devices (0 without a GPU; the library must still load)."""
    return int(_lib.load(require_device=False).hafb_device_count())


def _device(device) -> int:
    return int(os.environ.get("HAFB200_DEVICE", "0")) if device is None else int(device)


def sum_subsets_det(atilde, diag, n_half, backend, include_loops, workers, n_ranges,
                    cap_mult=SWEEP_CAP_MULT, *, arith=None, device=None):
    """Per-range Kahan partials (c128[n_ranges], int64[n_ranges]); ``workers`` does
    not change the result (the reference's deterministic contract), so it is
    only validated.  Replaces _numba.py:354-384."""
    lib = _lib.load(require_device=True)
    at, dg = _lib.c128(atilde), _lib.c128(diag)
    sums = np.zeros(n_ranges, np.complex128)
    fails = np.zeros(n_ranges, np.int64)
    _lib.check(lib.hafb_sum_subsets_det(_lib.dptr(at), _lib.dptr(dg), int(n_half), int(backend),
                                        int(bool(include_loops)), int(n_ranges), int(cap_mult),
                                        _arith_id(arith), _device(device), _lib.dptr(sums),
                                        _lib.i64ptr(fails)))
    return sums, fails


def sum_subsets_fast(atilde, diag, n_half, backend, include_loops, workers, n_ranges,
                     cap_mult=SWEEP_CAP_MULT, *, arith=None, device=None):
    """Per-worker compensated sums (c128[workers], int64[workers]) with the
    reference's range-to-worker dealing.  Replaces _numba.py:387-412."""
    lib = _lib.load(require_device=True)
    at, dg = _lib.c128(atilde), _lib.c128(diag)
    sums = np.zeros(workers, np.complex128)
    fails = np.zeros(workers, np.int64)
    _lib.check(lib.hafb_sum_subsets_fast(_lib.dptr(at), _lib.dptr(dg), int(n_half), int(backend),
                                         int(bool(include_loops)), int(workers), int(n_ranges),
                                         int(cap_mult), _arith_id(arith), _device(device),
                                         _lib.dptr(sums), _lib.i64ptr(fails)))
    return sums, fails


def sum_mask_range(atilde, diag, n_half, lo, hi, n_chunks, backend, include_loops,
                   cap_mult=SWEEP_CAP_MULT, *, arith=None, device=None):
    """Kahan partials of masks [lo, hi) in n_chunks equal chunks (mask 0 skipped):
    the identical-range harness of SURVEY.md 8(c) for n >= 48."""
    lib = _lib.load(require_device=True)
    at, dg = _lib.c128(atilde), _lib.c128(diag)
    sums = np.zeros(n_chunks, np.complex128)
    fails = np.zeros(n_chunks, np.int64)
    _lib.check(lib.hafb_sum_mask_range(_lib.dptr(at), _lib.dptr(dg), int(n_half), int(lo), int(hi),
                                       int(n_chunks), int(backend), int(bool(include_loops)),
                                       int(cap_mult), _arith_id(arith), _device(device),
                                       _lib.dptr(sums), _lib.i64ptr(fails)))
    return sums, fails


def sum_range_list(atilde, diag, n_half, n_ranges, ranges, backend, include_loops,
                   cap_mult=SWEEP_CAP_MULT, *, arith=None, device=None):
    """Partials of an explicit list of the standard ranges (multi-GPU shards)."""
    lib = _lib.load(require_device=True)
    at, dg = _lib.c128(atilde), _lib.c128(diag)
    rl = np.ascontiguousarray(ranges, dtype=np.int32)
    sums = np.zeros(rl.size, np.complex128)
    fails = np.zeros(rl.size, np.int64)
    _lib.check(lib.hafb_sum_range_list(_lib.dptr(at), _lib.dptr(dg), int(n_half), int(n_ranges),
                                       _lib.i32ptr(rl), int(rl.size), int(backend),
                                       int(bool(include_loops)), int(cap_mult), _arith_id(arith),
                                       _device(device), _lib.dptr(sums), _lib.i64ptr(fails)))
    return sums, fails


def terms(atilde, diag, n_half, masks, backend, include_loops, cap_mult=SWEEP_CAP_MULT, *,
          arith=None, device=None):
    """Signed terms of many masks at once (c128[count], int32[count])."""
    lib = _lib.load(require_device=True)
    at, dg = _lib.c128(atilde), _lib.c128(diag)
    mk = np.ascontiguousarray(masks, dtype=np.uint64)
    out = np.zeros(mk.size, np.complex128)
    st = np.zeros(mk.size, np.int32)
    _lib.check(lib.hafb_terms(_lib.dptr(at), _lib.dptr(dg), int(n_half), _lib.u64ptr(mk), mk.size,
                              int(backend), int(bool(include_loops)), int(cap_mult),
                              _arith_id(arith), _device(device), _lib.dptr(out), _lib.i32ptr(st)))
    return out, st


def subset_term(atilde, diag, mask, n_half, backend, include_loops, cap_mult=SWEEP_CAP_MULT, *,
                arith=None, device=None):
    """(term, status) of one nonempty mask.  Replaces _numba.py:297-351."""
    out, st = terms(atilde, diag, n_half, [mask], backend, include_loops, cap_mult, arith=arith,
                    device=device)
    return complex(out[0]), int(st[0])


def batch(atilde, diag, n_half, backend, include_loops, n_ranges, cap_mult=SWEEP_CAP_MULT, *,
          arith=None, device=None):
    """Many prepared problems of one size: (c128[B], int64[B]) hafnians + statuses."""
    lib = _lib.load(require_device=True)
    at, dg = _lib.c128(atilde), _lib.c128(diag)
    B = at.shape[0]
    res = np.zeros(B, np.complex128)
    fails = np.zeros(B, np.int64)
    _lib.check(lib.hafb_batch(_lib.dptr(at), _lib.dptr(dg), int(B), int(n_half), int(backend),
                              int(bool(include_loops)), int(n_ranges), int(cap_mult),
                              _arith_id(arith), _device(device), _lib.dptr(res),
                              _lib.i64ptr(fails)))
    return res, fails


def batch_raw(a, n_half, backend, include_loops, n_ranges, symmetry_rtol,
              cap_mult=SWEEP_CAP_MULT, *, arith=None, device=None):
    """Raw matrices (B, n, n): device-side input semantics, then hafb_batch.
    Returns (results, fails, asym) with asym = None or (index, dev, tol)."""
    lib = _lib.load(require_device=True)
    A = _lib.c128(a)
    B = A.shape[0]
    res = np.zeros(B, np.complex128)
    fails = np.zeros(B, np.int64)
    idx = np.full(1, -1, np.int64)
    dev = np.zeros(1)
    tol = np.zeros(1)
    _lib.check(lib.hafb_batch_raw(_lib.dptr(A), int(B), int(n_half), int(backend),
                                  int(bool(include_loops)), int(n_ranges), int(cap_mult),
                                  _arith_id(arith), _device(device), float(symmetry_rtol),
                                  _lib.dptr(res), _lib.i64ptr(fails), _lib.i64ptr(idx),
                                  _lib.dptr(dev), _lib.dptr(tol)))
    asym = None if idx[0] < 0 else (int(idx[0]), float(dev[0]), float(tol[0]))
    return res, fails, asym


def power_traces_spectral(b, K, cap_mult=SWEEP_CAP_MULT, *, device=None):
    """(traces, sweeps, converged); destroys nothing (the device works on a copy).
    Replaces _numba.py:415-422: sweeps is the QR sweep count of the device iteration
    (identical to the reference's, which it replays operation for operation)."""
    lib = _lib.load(require_device=True)
    h = _lib.c128(b)
    out = np.zeros(K, np.complex128)
    sw = np.zeros(1, np.int64)
    ok = np.zeros(1, np.int32)
    _lib.check(lib.hafb_power_traces(_lib.dptr(h), h.shape[0], int(K), 0, int(cap_mult), 0,
                                     _device(device), _lib.dptr(out), _lib.i64ptr(sw),
                                     _lib.i32ptr(ok)))
    return out, int(sw[0]), bool(ok[0])


def power_traces_charpoly(b, K, *, device=None):
    """(traces, finite_ok).  Replaces _numba.py:425-433."""
    lib = _lib.load(require_device=True)
    h = _lib.c128(b)
    out = np.zeros(K, np.complex128)
    sw = np.zeros(1, np.int64)
    ok = np.zeros(1, np.int32)
    _lib.check(lib.hafb_power_traces(_lib.dptr(h), h.shape[0], int(K), 1, SWEEP_CAP_MULT, 0,
                                     _device(device), _lib.dptr(out), _lib.i64ptr(sw),
                                     _lib.i32ptr(ok)))
    return out, bool(ok[0])


def charpoly_coefficients(b, *, device=None):
    """Monic characteristic polynomial, ascending.  Replaces _numba.py:436-440."""
    lib = _lib.load(require_device=True)
    h = _lib.c128(b)
    out = np.zeros(h.shape[0] + 1, np.complex128)
    _lib.check(lib.hafb_charpoly_coefficients(_lib.dptr(h), h.shape[0], 0, _device(device),
                                              _lib.dptr(out)))
    return out


def modp_sums(atilde_p, diag_p, primes, n_half, lo, hi, include_loops, *, device=None):
    """Exact-mode residues: the signed subset sum over masks [lo, hi) modulo each
    prime (hafb_modp_sums).  atilde_p / diag_p: residues, one slice per prime.
    Returns (uint64[n_primes] residues, device milliseconds of the term kernels)."""
    lib = _lib.load(require_device=True)
    pr = np.ascontiguousarray(primes, dtype=np.uint32)
    at = np.ascontiguousarray(atilde_p, dtype=np.uint32)
    dg = np.ascontiguousarray(diag_p, dtype=np.uint32)
    n = 2 * int(n_half)
    if at.size != pr.size * n * n or dg.size != pr.size * n:
        raise ValueError("residue arrays do not match n_primes x n x n / n_primes x n")
    res = np.zeros(pr.size, np.uint64)
    ms = ctypes.c_double(0.0)
    u32 = ctypes.POINTER(ctypes.c_uint32)
    _lib.check(lib.hafb_modp_sums(at.ctypes.data_as(u32), dg.ctypes.data_as(u32),
                                  pr.ctypes.data_as(u32), int(pr.size), int(n_half), int(lo),
                                  int(hi), int(bool(include_loops)), _device(device),
                                  _lib.u64ptr(res), ctypes.byref(ms)))
    return res, ms.value
