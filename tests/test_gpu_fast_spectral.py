"""FAST arithmetic on the spectral backend (csrc/qr_fast.cuh): the reference's shifted
QR (_numba.py:70-188) and power sums (:191-200) in FMA arithmetic on the FAST kernel's
packed Hessenberg form; the 64-lane shared-memory sizes (S >= 40, or S >= 34 with
loops) keep the bit-exact QR kernel.

Checked per term against the bit-exact oracle's spectral terms at every size class,
and whole problems against the extended-precision referee with the accuracy contract
of paper_1805_12498_b200/accuracy.py (|x - truth| <= max(1e-10 |truth|, 5e-15 sum|t|)).
Non-convergence keeps the reference's status 1 -> EigensolverNoConvergence.
"""

import numpy as np
import pytest

from conftest import has_gpu, load_golden, random_symmetric
from oracle import oracle as O
from paper_1805_12498_b200 import accuracy, engine, kernels
from paper_1805_12498_b200.errors import EigensolverNoConvergence

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


def _sample_masks(nh, S, count, seed):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        bits = rng.choice(nh, size=S // 2, replace=False)
        out.append(int(sum(1 << int(b) for b in bits)))
    return np.array(out, dtype=np.uint64)


@pytest.mark.parametrize("S", [2, 4, 6, 8, 12, 16, 18, 22, 26, 30, 32, 34, 36, 38, 40, 44])
@pytest.mark.parametrize("loops", [False, True])
def test_fast_spectral_terms_every_size_vs_oracle(S, loops):
    """Per-term FAST spectral vs the bit-exact oracle (spectral backend) for sampled
    subsets of one size class; tolerance relative to the class's largest term."""
    n = max(S, 20) + (max(S, 20) % 2)
    A = random_symmetric(n, 3000 + S) / np.sqrt(n)
    if loops:
        np.fill_diagonal(A, np.random.default_rng(S).normal(size=n) * 0.5)
    at, dg, nh = engine._prepare(A, loops)
    masks = _sample_masks(nh, S, 12, 40 + S)
    ref, rst = O.terms(at, dg, nh, masks, backend=0, include_loops=loops)
    got, st = kernels.terms(at, dg, nh, masks, 0, loops, arith="fast")
    assert np.array_equal(st, rst)
    scale = np.abs(ref).max()
    assert np.abs(got - ref).max() <= 1e-9 * scale, np.abs(got - ref).max() / scale


@pytest.mark.parametrize("name", ["cfg0", "cfg2", "cfg3", "cfg1s0", "cfg1s1"])
def test_fast_spectral_whole_problem_vs_referee(name):
    """Whole problems through the public API with backend="spectral", arith="fast"
    (cfg2 is the loop hafnian), against the referee's truth."""
    ref = load_golden("referee.npz")
    c = load_golden("ranges.npz")[name]
    loops = bool(c["loops"])
    f = engine.loop_hafnian if loops else engine.hafnian
    got = f(c["A"], backend="spectral", arith="fast")
    hi, lo, sa = complex(ref[name]["hi"]), complex(ref[name]["lo"]), float(ref[name]["abs_sum"])
    assert accuracy.within(got, hi, lo, sa), (name, accuracy.error(got, hi, lo) / abs(hi))


def test_fast_spectral_n52_range_vs_referee():
    """North-star identical range [0, 2^16) of the n = 52 input on the spectral backend:
    FAST within the contract, and the bit-exact MIRROR spectral result for reference."""
    case = load_golden("range_n52.npz")["n52s3"]
    at, dg, nh = engine._prepare(case["A"], False)
    s_fast, f_fast = kernels.sum_mask_range(at, dg, nh, 0, 1 << 16, 512, 0, False, arith="fast")
    s_mir, f_mir = kernels.sum_mask_range(at, dg, nh, 0, 1 << 16, 512, 0, False, arith="mirror")
    assert not f_fast.any() and not f_mir.any()
    r_fast, r_mir = engine.tree_reduce(s_fast), engine.tree_reduce(s_mir)
    masks = np.arange(1, 1 << 16, dtype=np.uint64)
    t, _ = kernels.terms(at, dg, nh, masks, 0, False, arith="fast")
    sa = float(np.abs(t).sum())
    # both are double-precision evaluations of the same value: within the contract's
    # rounding-level bound of each other
    assert abs(r_fast - r_mir) <= 2 * accuracy.bound(r_mir, sa)


def test_fast_spectral_sweep_cap_zero_raises(monkeypatch):
    """cap 0: the first sweep is refused (status 1), as in the reference."""
    monkeypatch.setattr(kernels, "SWEEP_CAP_MULT", 0)
    a = random_symmetric(12, 15)
    np.fill_diagonal(a, 0)
    with pytest.raises(EigensolverNoConvergence):
        engine.hafnian(a, backend="spectral", arith="fast")


def test_fast_spectral_agrees_with_fast_charpoly():
    """The two FAST backends compute the same term by different routes (eigenvalues vs
    characteristic polynomial): per-term agreement on a random n = 30 problem."""
    A = random_symmetric(30, 77) / np.sqrt(30)
    at, dg, nh = engine._prepare(A, False)
    masks = np.arange(1, 1 << 15, 7, dtype=np.uint64)
    ts, ss = kernels.terms(at, dg, nh, masks, 0, False, arith="fast")
    tc, sc = kernels.terms(at, dg, nh, masks, 1, False, arith="fast")
    assert not ss.any() and not sc.any()
    assert np.abs(ts - tc).max() <= 1e-9 * np.abs(tc).max()
