"""The reference's kernel-module contract as a drop-in plugin module.

``hafnium.kernels.active()`` (pkg/src/hafnium/kernels/__init__.py:53-56) returns a
module with exactly these names; ``hafnium.engine._compute`` (engine.py:153-178)
and ``engine.subset_term`` (:198-216) call them positionally and read
``SWEEP_CAP_MULT`` from the module at call time.  INTEGRATION.md §2 installs this
module as ``hafnium/kernels/_b200.py`` (a one-line re-export) behind
``HAFNIUM_KERNELS=b200``.

Arithmetic: ``HAFB200_ARITH`` (read per call; default "mirror") picks MIRROR
(bit-identical to the numba kernels) or FAST (FMA-contracted, within the
rounding-level bound of accuracy.py) for both backends: FAST spectral runs the
reference's shifted QR in FMA arithmetic (csrc/qr_fast.cuh).
"""

from __future__ import annotations

from . import kernels as _k

SWEEP_CAP_MULT = 30  # _numba.py:33; monkeypatchable like the reference's


def sum_subsets_det(atilde, diag, n_half, backend, include_loops, workers, n_ranges, cap_mult):
    """_numba.py:354-384."""
    return _k.sum_subsets_det(atilde, diag, n_half, backend, include_loops, workers, n_ranges,
                              cap_mult, arith=_k.default_arith())


def sum_subsets_fast(atilde, diag, n_half, backend, include_loops, workers, n_ranges, cap_mult):
    """_numba.py:387-412."""
    return _k.sum_subsets_fast(atilde, diag, n_half, backend, include_loops, workers, n_ranges,
                               cap_mult, arith=_k.default_arith())


def subset_term(atilde, diag, mask, n_half, backend, include_loops, cap_mult):
    """_numba.py:297-351."""
    return _k.subset_term(atilde, diag, mask, n_half, backend, include_loops, cap_mult,
                          arith=_k.default_arith())


def power_traces_spectral(b, K, cap_mult):
    """_numba.py:415-422: (traces, sweeps, converged)."""
    return _k.power_traces_spectral(b, K, cap_mult)


def power_traces_charpoly(b, K):
    """_numba.py:425-433: (traces, ok)."""
    return _k.power_traces_charpoly(b, K)


def charpoly_coefficients(b):
    """_numba.py:436-440."""
    return _k.charpoly_coefficients(b)
