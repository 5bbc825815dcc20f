"""Parity of the device path (through the C ABI) with the reference.

MIRROR arithmetic reproduces the reference's IEEE operation sequence, so its
terms, range partials and totals are compared BIT-EXACTLY with fixtures
produced by the reference itself (tests/golden) and with the C oracle.
FAST arithmetic is compared within the stated tolerances.
"""

import itertools

import numpy as np
import pytest

from conftest import bits, has_gpu, load_golden, random_symmetric, rel_err
from oracle import bruteforce as BF
from oracle import oracle as O
from paper_1805_12498_b200 import engine, kernels, workloads
from paper_1805_12498_b200.errors import DegenerateHessenberg, OddDimension

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


# ------------------------------------------------------------------ golden, bit-exact

def test_terms_mirror_bit_exact_vs_reference():
    g = load_golden("terms.npz")
    for name, case in g.items():
        loops = bool(case["loops"])
        at, dg, nh = engine._prepare(case["A"], loops)
        for backend in (1, 0):
            vals, st = kernels.terms(at, dg, nh, case["masks"], backend, loops, arith="mirror")
            assert np.array_equal(st, case[f"status_b{backend}"]), name
            same = bits(vals) == bits(case[f"terms_b{backend}"])
            assert same.all(), f"{name} b{backend}: {np.count_nonzero(~same)} words differ"


def test_range_partials_mirror_bit_exact_vs_reference():
    g = load_golden("ranges.npz")
    for name, case in g.items():
        loops = bool(case["loops"])
        at, dg, nh = engine._prepare(case["A"], loops)
        nr = min((1 << nh) - 1, 512)
        for backend in (1, 0):
            sums, fails = kernels.sum_subsets_det(at, dg, nh, backend, loops, 1, nr, arith="mirror")
            assert (bits(sums) == bits(case[f"partials_b{backend}"])).all(), f"{name} b{backend}"
            assert np.array_equal(fails, case[f"fails_b{backend}"])
            fs, _ = kernels.sum_subsets_fast(at, dg, nh, backend, loops, 3, nr, arith="mirror")
            assert (bits(fs) == bits(case[f"fast3_b{backend}"])).all(), f"{name} fast b{backend}"


def test_public_api_bit_identical_to_reference_results():
    g = load_golden("ranges.npz")
    for name, case in g.items():
        loops = bool(case["loops"])
        f = engine.loop_hafnian if loops else engine.hafnian
        for backend, bname in ((1, "charpoly"), (0, "spectral")):
            got = f(case["A"], backend=bname)
            assert got == complex(case[f"result_b{backend}"]), (name, bname)


def test_cfg3_matching_count_rounds_like_reference():
    """cfg3 (n=40 ER graph): the mirror result equals the reference's float result,
    so rounding it gives the reference's integer; the exact count differs from both
    (the float formula cannot resolve 3.1e17 > 2^53, SURVEY.md finding 4)."""
    g = load_golden("ranges.npz")["cfg3"]
    got = engine.hafnian(g["A"], backend="charpoly")
    assert got == complex(g["result_b1"])
    assert round(got.real) == round(complex(g["result_b1"]).real)
    exact = 308544357990268074
    assert abs(got.real - exact) / exact < 1e-5


def test_n52_range_mirror_bit_exact():
    g = load_golden("range_n52.npz")
    for name, case in g.items():
        at, dg, nh = engine._prepare(case["A"], False)
        for backend in (1, 0):
            key = f"partials_b{backend}"
            if key not in case:
                continue
            sums, fails = kernels.sum_mask_range(at, dg, nh, 0, 1 << 20, 512, backend, False,
                                                 arith="mirror")
            assert (bits(sums) == bits(case[key])).all(), (name, backend)
            assert engine.tree_reduce(sums) == complex(case[f"result_b{backend}"])


def test_batch_equals_single_calls():
    g = load_golden("ranges.npz")
    mats = [g[f"cfg1s{s}"]["A"] for s in range(4)]
    res = engine.hafnian_batch(mats, backend="charpoly")
    for s in range(4):
        assert res[s] == complex(g[f"cfg1s{s}"]["result_b1"])
    res0 = engine.hafnian_batch(mats, backend="spectral")
    for s in range(4):
        assert res0[s] == complex(g[f"cfg1s{s}"]["result_b0"])


def test_batch_device_input_semantics():
    """hafnian_batch runs matrix.py's strict check + mirror and engine._prepare on the
    device: same bits as the single-matrix path (which does them on the host), same
    AsymmetricInput decision and message, loops and non-finite inputs included."""
    from paper_1805_12498_b200.errors import AsymmetricInput

    rng = np.random.default_rng(11)
    mats = []
    for b in range(6):
        a = random_symmetric(12, 500 + b)
        i, j = rng.integers(0, 12, 2)
        if i != j:  # upper/lower differ within tolerance: the upper triangle must win
            a[min(i, j), max(i, j)] += 1e-13
        mats.append(a)
    mats = np.stack(mats)
    for loops, f in ((False, engine.hafnian), (True, engine.loop_hafnian)):
        for arith in ("mirror", "fast"):
            res = engine.hafnian_batch(mats, backend="charpoly", arith=arith, loops=loops)
            for b in range(len(mats)):
                assert res[b] == f(mats[b], backend="charpoly", arith=arith), (loops, arith, b)
    bad = mats.copy()
    bad[3, 0, 5] += 1e-6
    with pytest.raises(AsymmetricInput) as e1:
        engine.hafnian_batch(bad)
    with pytest.raises(AsymmetricInput) as e2:
        engine.hafnian(bad[3])
    assert str(e1.value).startswith("matrix 3: ")
    assert str(e1.value)[len("matrix 3: "):] == str(e2.value)
    nanm = mats.copy()
    nanm[1, 2, 2] = np.nan  # numpy: NaN deviation never exceeds the tolerance
    r, fails, asym = kernels.batch_raw(nanm, 6, 1, True, 63, 1e-12)
    assert asym is None
    at, dg, nh = engine._prepare(nanm[1], True)
    s1, f1 = kernels.sum_subsets_det(at, dg, nh, 1, True, 1, 63)
    assert fails[1] == f1.max()


def test_powertraces_mirror_bit_exact():
    g = load_golden("powertraces.npz")
    for q, case in g.items():
        b, K = case["b"], int(case["K"])
        t, ok = kernels.power_traces_charpoly(b, K)
        assert ok == bool(case["charpoly_ok"])
        assert (bits(t) == bits(case["charpoly_traces"])).all(), q
        assert (bits(kernels.charpoly_coefficients(b)) == bits(case["coeffs"])).all(), q
        ts, sweeps, conv = kernels.power_traces_spectral(b, K)
        assert conv == bool(case["spectral_conv"])
        assert sweeps == int(case["spectral_sweeps"]), q  # the QR sweep count (_numba.py:415-422)
        assert (bits(ts) == bits(case["spectral_traces"])).all(), q


# ------------------------------------------------------------------ oracle, bit-exact

@pytest.mark.parametrize("n,loops,seed", [(2, False, 1), (6, True, 2), (16, False, 3),
                                          (18, True, 4), (24, False, 5), (28, True, 6)])
def test_random_vs_oracle_bit_exact(n, loops, seed):
    A = random_symmetric(n, seed)
    at, dg, nh = engine._prepare(A, loops)
    nr = min((1 << nh) - 1, 512)
    for backend in (1, 0):
        sums, fails = kernels.sum_subsets_det(at, dg, nh, backend, loops, 1, nr)
        ref, rf = O.sum_subsets_det(at, dg, nh, backend, loops, 8, nr)
        assert (bits(sums) == bits(ref)).all()
        assert np.array_equal(fails, rf)


def test_sharded_range_lists_reassemble_bit_exact():
    A = workloads.cfg0()
    at, dg, nh = engine._prepare(A, False)
    full, _ = kernels.sum_subsets_det(at, dg, nh, 1, False, 1, 512)
    from paper_1805_12498_b200 import costmodel

    for k in (2, 3, 8):
        shards = costmodel.lpt_shards(costmodel.range_costs(nh, 512), k)
        got = np.zeros(512, np.complex128)
        for sh in shards:
            s, f = kernels.sum_range_list(at, dg, nh, 512, sh, 1, False)
            got[sh] = s
        assert (bits(got) == bits(full)).all()


# ------------------------------------------------------------------ reference test KATs
# (the hot-path rows of SURVEY.md section 4, ported to the device API)

def test_empty_and_odd():
    assert engine.hafnian(np.zeros((0, 0))) == 1
    with pytest.raises(OddDimension):
        engine.hafnian(np.zeros((3, 3)))
    with pytest.raises(OddDimension):
        engine.loop_hafnian(np.eye(5))


def test_single_pair_and_4x4():
    a = 0.7 - 0.2j
    assert rel_err(engine.hafnian(np.array([[0, a], [a, 0]])), a) < 1e-14
    b = random_symmetric(4, 100)
    np.fill_diagonal(b, 0)
    expected = b[0, 1] * b[2, 3] + b[0, 2] * b[1, 3] + b[0, 3] * b[1, 2]
    assert rel_err(engine.hafnian(b), expected) < 1e-12


def test_diagonal_ignored_bitwise():
    a = random_symmetric(6, 101)
    b = a.copy()
    np.fill_diagonal(b, 0)
    assert engine.hafnian(a) == engine.hafnian(b)


@pytest.mark.parametrize("arith", ["mirror", "fast"])
def test_complete_graph_double_factorial(arith):
    a = np.ones((20, 20), dtype=complex)
    np.fill_diagonal(a, 0)
    for backend in ("charpoly", "spectral"):
        assert rel_err(engine.hafnian(a, backend=backend, arith=arith), BF.double_factorial(19)) < 1e-9


@pytest.mark.parametrize("m", [2, 3, 4, 5])
def test_bipartite_equals_permanent(m):
    rng = np.random.default_rng(m + 200)
    w = rng.uniform(-1, 1, (m, m)) + 1j * rng.uniform(-1, 1, (m, m))
    assert rel_err(engine.hafnian(BF.bipartite_embedding(w)), BF.permanent_ryser(w)) < 1e-9


@pytest.mark.parametrize("n", [2, 4, 6, 8, 10])
@pytest.mark.parametrize("arith", ["mirror", "fast"])
def test_random_vs_bruteforce(n, arith):
    a = random_symmetric(n, n + 300)
    np.fill_diagonal(a, 0)
    assert rel_err(engine.hafnian(a, backend="charpoly", arith=arith), BF.hafnian_bruteforce(a)) < 1e-10
    b = random_symmetric(n, n + 400)
    assert rel_err(engine.loop_hafnian(b, backend="charpoly", arith=arith),
                   BF.loop_hafnian_bruteforce(b)) < 1e-10


def test_loop_hafnian_kats():
    assert rel_err(engine.loop_hafnian(np.ones((10, 10))), BF.telephone(10)) < 1e-9
    d = np.array([1.5, -2.0, 0.5 + 1j, 3.0, -0.25, 2.0 - 1j])
    assert rel_err(engine.loop_hafnian(np.diag(d)), d.prod()) < 1e-12
    a = random_symmetric(10, 103)
    np.fill_diagonal(a, 0)
    assert engine.loop_hafnian(a) == engine.hafnian(a)


@pytest.mark.parametrize("n", [4, 6, 8, 10])
def test_matching_count_identity(n):
    rng = np.random.default_rng(n + 50)
    adj = np.triu((rng.uniform(size=(n, n)) < 0.6).astype(int), 1)
    adj = adj + adj.T
    count = BF.matching_count(adj)
    lhaf = engine.loop_hafnian(adj.astype(complex) + np.eye(n))
    assert round(lhaf.real) == count
    assert abs(lhaf - count) <= 1e-9 * max(1, count)


@pytest.mark.parametrize("mu", [0.5, 2.0, 3 + 4j])
@pytest.mark.parametrize("n", [4, 8, 12])
def test_homogeneity(mu, n):
    a = random_symmetric(n, n + 500)
    np.fill_diagonal(a, 0)
    assert rel_err(engine.hafnian(mu * a), mu ** (n // 2) * engine.hafnian(a)) < 1e-10


def test_subset_terms():
    a = 1.3 + 0.4j
    assert rel_err(engine.subset_term(np.array([[0, a], [a, 0]]), 1), a) < 1e-14
    k4 = np.ones((4, 4), dtype=complex)
    np.fill_diagonal(k4, 0)
    assert rel_err(sum(engine.subset_term(k4, m) for m in range(1, 4)), 3) < 1e-12
    with pytest.raises(ValueError):
        engine.subset_term(np.zeros((2, 2)), 0)
    with pytest.raises(ValueError):
        engine.subset_term(np.zeros((2, 2)), 2)


def test_deterministic_across_devices_and_repeats():
    a = np.ones((20, 20), dtype=complex)
    np.fill_diagonal(a, 0)
    results = {engine.hafnian(a, threads=t) for t in (1, 2, 4, 8)}
    assert len(results) == 1
    b = random_symmetric(12, 14)
    assert engine.hafnian(b) == engine.hafnian(b)


def test_concurrent_calls():
    import threading

    mats = [random_symmetric(10, 600 + i) for i in range(4)]
    expected = [engine.hafnian(m) for m in mats]
    out = [None] * 4

    def work(i):
        out[i] = engine.hafnian(mats[i], threads=2)

    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert out == expected


def test_sweep_cap_zero_raises(monkeypatch):
    from paper_1805_12498_b200.errors import EigensolverNoConvergence

    monkeypatch.setattr(kernels, "SWEEP_CAP_MULT", 0)
    a = random_symmetric(8, 15)
    np.fill_diagonal(a, 0)
    with pytest.raises(EigensolverNoConvergence):
        engine.hafnian(a)


def test_nonfinite_input_statuses_match_oracle():
    a = random_symmetric(8, 16)
    a[0, 1] = a[1, 0] = np.inf
    at, dg, nh = engine._prepare(a, False)
    for backend in (1, 0):
        _, fails = kernels.sum_subsets_det(at, dg, nh, backend, False, 1, 15)
        _, rf = O.sum_subsets_det(at, dg, nh, backend, False, 1, 15)
        assert np.array_equal(fails, rf)
    if O.sum_subsets_det(at, dg, nh, 1, False, 1, 15)[1].max() == 2:
        with pytest.raises(DegenerateHessenberg):
            engine.hafnian(a, backend="charpoly")


# ------------------------------------------------------------------ fast arithmetic

# FAST against the truth (the extended-precision referee): tests/test_gpu_referee.py


@pytest.mark.parametrize("S", [2, 4, 8, 12, 16, 18, 22, 26, 30, 32, 34, 38, 42, 46, 50])
def test_fast_terms_every_size_vs_oracle(S):
    """Per-term FAST vs the bit-exact oracle for subsets of every size class."""
    n = max(S, 20) + (max(S, 20) % 2)
    A = random_symmetric(n, 1000 + S) / np.sqrt(n)
    at, dg, nh = engine._prepare(A, False)
    rng = np.random.default_rng(S)
    masks = []
    for _ in range(16):
        bits = rng.choice(nh, size=S // 2, replace=False)
        masks.append(int(sum(1 << int(b) for b in bits)))
    masks = np.array(masks, dtype=np.uint64)
    ref, _ = O.terms(at, dg, nh, masks, backend=1)
    got, st = kernels.terms(at, dg, nh, masks, 1, False, arith="fast")
    scale = np.abs(ref).max()
    assert not st.any()
    assert np.abs(got - ref).max() <= 1e-10 * scale


@pytest.mark.parametrize("S", [34, 36, 38])
def test_fast_extra_row_classes_full_class_vs_oracle(S):
    """S = 34..38 run one-warp teams with the rows beyond 32 held column-wise (NSX).
    Every subset of the class for n = 44 (C(22, S/2) masks, thousands of teams walking
    long mask runs): no failing status, every term within 1e-10 of the largest oracle
    term, and a seeded sample checked per term against the bit-exact oracle."""
    n = 44
    A = random_symmetric(n, 2000 + S) / np.sqrt(n)
    at, dg, nh = engine._prepare(A, False)
    masks = np.array([sum(1 << b for b in c) for c in itertools.combinations(range(nh), S // 2)],
                     dtype=np.uint64)
    got, st = kernels.terms(at, dg, nh, masks, 1, False, arith="fast")
    assert not st.any()
    assert np.isfinite(got).all()
    idx = np.random.default_rng(S).choice(masks.size, 1500, replace=False)
    ref, _ = O.terms(at, dg, nh, masks[idx], backend=1)
    scale = np.abs(ref).max()
    assert np.abs(got[idx] - ref).max() <= 1e-10 * scale


@pytest.mark.parametrize("n", [52, 60])
@pytest.mark.parametrize("symmetric", [True, False])
def test_fast_triangular_staging_and_asymmetric_fallback(n, symmetric):
    """The split-row NSX classes (S = 34, 36) run 12 teams per SM; where the full staged
    Atilde no longer fits beside them the blocks stage only the lower triangle of the
    symmetric A behind Atilde = X A, after verifying Atilde[r][c] == Atilde[c^1][r^1] bit for
    bit.  An Atilde that is not of that form (legal at the kernel-module contract, which takes
    any matrix) must take the global-memory gather instead and still match the oracle."""
    A = random_symmetric(n, 4242 + n) / np.sqrt(n)
    at, dg, nh = engine._prepare(A, False)
    if not symmetric:
        rng = np.random.default_rng(n)
        at = at + 1e-3 * (rng.normal(size=at.shape) + 1j * rng.normal(size=at.shape))
    rng = np.random.default_rng(7 * n)
    masks = []
    for S in (30, 32, 34, 36):
        for _ in range(24):
            bits = rng.choice(nh, size=S // 2, replace=False)
            masks.append(int(sum(1 << int(b) for b in bits)))
    masks = np.array(masks, dtype=np.uint64)
    ref, _ = O.terms(at, dg, nh, masks, backend=1)
    got, st = kernels.terms(at, dg, nh, masks, 1, False, arith="fast")
    assert not st.any()
    for k in range(4):  # per size class: terms of different classes differ by orders of magnitude
        sl = slice(24 * k, 24 * (k + 1))
        assert np.abs(got[sl] - ref[sl]).max() <= 1e-10 * np.abs(ref[sl]).max()


@pytest.mark.parametrize("n", [34, 36, 38])
def test_fast_nsx_whole_problems(n):
    """Whole problems whose largest classes run on the NSX kernel: FAST vs the bit-exact
    MIRROR result (= the reference), on a Gaussian matrix scaled like the bench input
    and in a batch (several problems per launch: staged and global gathers)."""
    rng = np.random.default_rng(n)
    g = rng.normal(0, np.sqrt(0.5), (n, n)) + 1j * rng.normal(0, np.sqrt(0.5), (n, n))
    a = (g + g.T) / 2 / np.sqrt(n)
    ref = engine.hafnian(a, backend="charpoly", arith="mirror")
    got = engine.hafnian(a, backend="charpoly", arith="fast")
    at, dg, nh = engine._prepare(a, False)
    t, _ = kernels.terms(at, dg, nh, np.arange(1, 1 << nh, dtype=np.uint64), 1, False, arith="fast")
    abs_sum = float(np.abs(t).sum())
    assert abs(got - ref) <= max(1e-10 * abs(ref), 1e-15 * abs_sum), (abs(got - ref) / abs(ref))
    b = engine.hafnian_batch(np.stack([a, a.T.copy(), 2 * a]), backend="charpoly", arith="fast")
    assert np.allclose(b, [got, got, got * 2 ** (n // 2)], rtol=1e-12, atol=0)


def test_fast_nsx_zero_columns_counting():
    """A 0/1 adjacency matrix at n = 36 (exactly zero pivot columns occur in the
    reduction): FAST against the exact GF(p) count, under the stated FAST tolerance
    max(1e-10 |ref|, 1e-15 sum|t|).  This input cancels by sum|t|/count ~ 7e8: FAST
    lands 1.8e-8 from the count, the reference's own arithmetic (MIRROR) 8.0e-8."""
    from paper_1805_12498_b200 import exact
    rng = np.random.default_rng(7)
    adj = np.triu((rng.uniform(size=(36, 36)) < 0.3).astype(np.int64), 1)
    a = adj + adj.T
    count = exact.hafnian_exact(a)
    ac = a.astype(np.complex128)
    got = engine.hafnian(ac, backend="charpoly", arith="fast")
    at, dg, nh = engine._prepare(ac, False)
    t, st = kernels.terms(at, dg, nh, np.arange(1, 1 << nh, dtype=np.uint64), 1, False, arith="fast")
    assert not st.any()
    abs_sum = float(np.abs(t).sum())
    assert abs(got - count) <= max(1e-10 * count, 1e-15 * abs_sum), (abs(got - count) / count)
    mirror = engine.hafnian(ac, backend="charpoly", arith="mirror")
    assert abs(got - count) <= abs(mirror - count)  # no worse than the reference here


@pytest.mark.parametrize("n", [60, 62])
def test_fast_terms_at_the_size_limit(n):
    """n = 60, 62 (D up to kDMax = 31): FAST terms of sampled masks from every class
    from S = 2 to S = n against the bit-exact oracle."""
    rng = np.random.default_rng(n)
    g = rng.normal(0, np.sqrt(0.5), (n, n)) + 1j * rng.normal(0, np.sqrt(0.5), (n, n))
    a = (g + g.T) / 2 / np.sqrt(n)
    at, dg, nh = engine._prepare(a, False)
    masks = []
    for m in range(1, nh + 1):
        for _ in range(3):
            bits = rng.choice(nh, size=m, replace=False)
            masks.append(int(sum(1 << int(b) for b in bits)))
    masks = np.array(masks, dtype=np.uint64)
    ref, rst = O.terms(at, dg, nh, masks, backend=1)
    got, st = kernels.terms(at, dg, nh, masks, 1, False, arith="fast")
    assert np.array_equal(st, rst)
    pc = np.array([bin(int(x)).count("1") for x in masks])
    for m in range(1, nh + 1):
        sel = pc == m
        scale = np.abs(ref[sel]).max()
        assert np.abs(got[sel] - ref[sel]).max() <= 1e-9 * scale, (m, np.abs(got[sel] - ref[sel]).max() / scale)


def test_fast_loop_terms_every_class_n40():
    """Loop-hafnian FAST terms (loop chain + Newton/exp path; static-column kernel up to
    S = 32, shared-memory kernel from S = 34) of sampled masks from every class of an
    n = 40 problem against the bit-exact oracle."""
    n = 40
    rng = np.random.default_rng(40)
    g = rng.normal(0, np.sqrt(0.5), (n, n)) + 1j * rng.normal(0, np.sqrt(0.5), (n, n))
    a = (g + g.T) / 2 / np.sqrt(n)
    np.fill_diagonal(a, rng.normal(0, np.sqrt(0.5), n) + 1j * rng.normal(0, np.sqrt(0.5), n))
    at, dg, nh = engine._prepare(a, True)
    masks = []
    for m in range(1, nh + 1):
        for _ in range(6):
            bits = rng.choice(nh, size=m, replace=False)
            masks.append(int(sum(1 << int(b) for b in bits)))
    masks = np.array(masks, dtype=np.uint64)
    ref, rst = O.terms(at, dg, nh, masks, backend=1, include_loops=True)
    got, st = kernels.terms(at, dg, nh, masks, 1, True, arith="fast")
    assert np.array_equal(st, rst)
    pc = np.array([bin(int(x)).count("1") for x in masks])
    for m in range(1, nh + 1):
        sel = pc == m
        scale = np.abs(ref[sel]).max()
        assert np.abs(got[sel] - ref[sel]).max() <= 1e-9 * scale, (m, np.abs(got[sel] - ref[sel]).max() / scale)


def test_fast_sharded_range_lists_reassemble_bit_exact_n36():
    """FAST range partials over LPT shards (many segments per launch: each team's contiguous
    mask walk crosses segment edges) equal the full run bit for bit at n = 36 (NSX, both
    static-column team widths, staged gathers)."""
    from paper_1805_12498_b200 import costmodel

    rng = np.random.default_rng(36)
    n = 36
    g = rng.normal(0, np.sqrt(0.5), (n, n)) + 1j * rng.normal(0, np.sqrt(0.5), (n, n))
    a = (g + g.T) / 2 / np.sqrt(n)
    at, dg, nh = engine._prepare(a, False)
    full, ff = kernels.sum_subsets_det(at, dg, nh, 1, False, 1, 512, arith="fast")
    assert not ff.any()
    for k in (3, 8):
        shards = costmodel.lpt_shards(costmodel.range_costs(nh, 512), k)
        got = np.zeros(512, np.complex128)
        for sh in shards:
            s, f = kernels.sum_range_list(at, dg, nh, 512, sh, 1, False, arith="fast")
            assert not f.any()
            got[sh] = s
        assert (bits(got) == bits(full)).all()
