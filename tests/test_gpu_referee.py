"""FAST and MIRROR on the device, scored against the extended-precision referee.

The referee (oracle/referee.c in x87 long double, checked against binary128 and
exact counts by tests/test_referee.py) gives each config's true value to ~2^-64
x cond.  MIRROR is bit-identical to the reference, so its error IS the
reference's.  Tolerance (paper_1805_12498_b200/accuracy.py, stated here once):

    |x - truth| <= max(1e-10 |truth|, 5e-15 sum|t|)

-- the bound the reference's own results meet on every config and that the plain
1e-10 relative bound is not (the reference misses it on cfg2, the n=56 range and
621 of the 4096 cfg1 matrices).  On the 4096-matrix batch FAST must also match the
reference's error DISTRIBUTION (quantiles within the stated factors).
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, digest, has_gpu, load_golden
from paper_1805_12498_b200 import accuracy, engine, kernels, workloads

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


def _truth(g, key):
    return complex(g[key]["hi"]), complex(g[key]["lo"]), float(g[key]["abs_sum"])


@pytest.mark.parametrize("name", ["cfg0", "cfg2", "cfg3", "cfg1s0", "cfg1s1", "cfg1s2", "cfg1s3"])
@pytest.mark.parametrize("arith", ["fast", "mirror"])
def test_whole_problem_vs_referee(name, arith):
    """Whole problems through the public API; cfg2 is the loop hafnian (FAST and MIRROR)."""
    ref = load_golden("referee.npz")
    c = load_golden("ranges.npz")[name]
    loops = bool(c["loops"])
    f = engine.loop_hafnian if loops else engine.hafnian
    got = f(c["A"], backend="charpoly", arith=arith)
    hi, lo, sa = _truth(ref, name)
    assert accuracy.within(got, hi, lo, sa), (name, arith, accuracy.error(got, hi, lo) / abs(hi))
    if arith == "mirror":
        assert got == complex(c["result_b1"])  # the reference's own value, bit for bit
    if name == "cfg3":  # the exact count: FAST is nearer to it than the reference
        exact = 308544357990268074
        assert abs(got.real - exact) <= abs(complex(c["result_b1"]).real - exact) or arith == "mirror"


@pytest.mark.parametrize("name", ["n52s3", "n52s4", "n56s4", "n64s5"])
def test_identical_range_vs_referee(name):
    """North-star parity for n >= 48: masks [0, 2^20) of the n=52 / n=56 inputs (seeds 3, 4)
    and of an n=64 input (seed 5; D = 32, the 32-bit-mask limit)."""
    ref = load_golden("referee.npz")
    case = load_golden("range_n64.npz" if name == "n64s5" else "range_n52.npz")[name]
    hi, lo, sa = _truth(ref, f"range_{name}")
    at, dg, nh = engine._prepare(case["A"], False)
    for arith in ("fast", "mirror"):
        sums, fails = kernels.sum_mask_range(at, dg, nh, 0, 1 << 20, 512, 1, False, arith=arith)
        assert not fails.any()
        got = engine.tree_reduce(sums)
        assert accuracy.within(got, hi, lo, sa), (name, arith, accuracy.error(got, hi, lo) / abs(hi))
        if arith == "mirror":
            assert got == complex(case["result_b1"])


def test_terms_vs_referee():
    """Per-term: FAST's worst relative error over every golden mask set is the
    reference's (within 2x overall, 4x + 1e-15 per case)."""
    ref = load_golden("referee.npz")
    worst_fast = worst_ref = 0.0
    for name, c in load_golden("terms.npz").items():
        loops = bool(c["loops"])
        at, dg, nh = engine._prepare(c["A"], loops)
        truth = ref[f"terms_{name}"]["values"]
        got, st = kernels.terms(at, dg, nh, c["masks"], 1, loops, arith="fast")
        assert not st.any()
        sc = np.maximum(np.abs(truth), 1e-300)
        ef = float(np.max(np.abs(got - truth) / sc))
        er = float(np.max(np.abs(c["terms_b1"] - truth) / sc))
        assert ef <= 4 * er + 1e-15, (name, ef, er)
        worst_fast, worst_ref = max(worst_fast, ef), max(worst_ref, er)
    assert worst_fast <= 2 * worst_ref, (worst_fast, worst_ref)


def _batch_inputs(count):
    G = np.load(os.path.join(GOLDEN, "batch_cfg1.npz"))
    As = np.array([workloads.cfg1(s) for s in range(count)])
    same = np.array([digest(a) for a in As], dtype=np.uint64) == G["digests"][:count]
    return G, As, same


def test_batch_cfg1_4096_mirror_bit_identical_to_reference():
    """The configured cfg1 workload: all 4096 GBS-like n=24 hafnians, MIRROR, against the
    reference's public-API results (tests/golden/batch_cfg1.npz, charpoly backend)."""
    G, As, same = _batch_inputs(4096)
    got = engine.hafnian_batch(As, backend="charpoly", arith="mirror")
    ref = G["result_b1"]
    assert same.mean() > 0.99  # inputs regenerate bit for bit (LAPACK QR is CPU-dependent)
    eq = got.view(np.uint64).reshape(-1, 2) == ref.view(np.uint64).reshape(-1, 2)
    assert eq[same].all(), np.count_nonzero(~eq[same].all(axis=1))


def test_batch_cfg1_4096_fast_vs_referee():
    """FAST on the 4096-matrix batch: every matrix within the rounding-level bound, and
    the error distribution is the reference's (median within 1.25x, p90/p99/max within
    2x, count above 1e-10 within 1.25x)."""
    B = np.load(os.path.join(GOLDEN, "referee_batch.npz"))
    G, As, same = _batch_inputs(4096)
    got = engine.hafnian_batch(As, backend="charpoly", arith="fast")
    hi, lo, sa = B["hi"][same], B["lo"][same], B["abs_sum"][same]
    ef = np.abs((got[same] - hi) - lo)
    er = np.abs((G["result_b1"][same] - hi) - lo)
    bound = np.maximum(accuracy.REL * np.abs(hi), accuracy.ABS_SUM * sa)
    assert (ef <= bound).all(), np.count_nonzero(ef > bound)
    rf, rr = ef / np.abs(hi), er / np.abs(hi)
    qf, qr = np.quantile(rf, [0.5, 0.9, 0.99, 1.0]), np.quantile(rr, [0.5, 0.9, 0.99, 1.0])
    assert qf[0] <= 1.25 * qr[0], (qf, qr)
    assert (qf[1:] <= 2 * qr[1:]).all(), (qf, qr)
    assert np.count_nonzero(rf > 1e-10) <= 1.25 * np.count_nonzero(rr > 1e-10)


def test_full_n52_vs_referee():
    """The headline workload itself: the FULL n=52 seed-3 hafnian (2^26-1 terms), FAST
    and MIRROR (== the reference's charpoly result), against the long double referee
    of the whole sum (tests/golden/referee_full52.npz)."""
    path = os.path.join(GOLDEN, "referee_full52.npz")
    if not os.path.exists(path):
        pytest.skip("referee_full52.npz not generated")
    R = np.load(path)
    hi, lo, sa = complex(R["hi"]), complex(R["lo"]), float(R["abs_sum"])
    A = R["A"]
    for arith in ("fast", "mirror"):
        got = engine.hafnian(A, backend="charpoly", arith=arith)
        assert accuracy.within(got, hi, lo, sa), (arith, accuracy.error(got, hi, lo) / abs(hi))


def test_n64_large_class_terms():
    """n = 64: sampled subsets of the large classes (S = 42..64, incl. the full mask),
    MIRROR bit-identical to the reference's terms, FAST within the reference's per-term
    error against the referee."""
    c = load_golden("range_n64.npz")["n64s5"]
    truth = load_golden("referee.npz")["terms_n64s5"]["values"]
    at, dg, nh = engine._prepare(c["A"], False)
    assert nh == 32
    mir, st = kernels.terms(at, dg, nh, c["masks"], 1, False, arith="mirror")
    assert not st.any()
    assert (mir.view(np.uint64) == c["terms_b1"].view(np.uint64)).all()
    fast, st = kernels.terms(at, dg, nh, c["masks"], 1, False, arith="fast")
    assert not st.any()
    sc = np.abs(truth)
    ef = np.max(np.abs(fast - truth) / sc)
    er = np.max(np.abs(c["terms_b1"] - truth) / sc)
    assert ef <= 4 * er + 1e-15, (ef, er)
