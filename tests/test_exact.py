"""Exact GF(p)+CRT mode: hafnian_exact / loop_hafnian_exact.

Checked against independent exact-integer oracles (oracle/bruteforce.py:
memoised matching DP with Python ints, closed forms (n-1)!! and T(n), Ryser's
permanent in exact ints) and the cfg3 known answer 308544357990268074
(SURVEY.md Appendix A).  Integer work: every comparison is exact equality.
"""

import numpy as np
import pytest

from conftest import has_gpu
from oracle.bruteforce import (
    bipartite_embedding,
    double_factorial,
    hafnian_exact_dp,
    telephone,
)
from paper_1805_12498_b200 import exact, kernels, workloads
from paper_1805_12498_b200.errors import AsymmetricInput, NonSquare, OddDimension, TooLarge

CFG3_EXACT = 308544357990268074


def _rand_int_sym(n, seed, lo=-9, hi=10, diag=True):
    rng = np.random.default_rng(seed)
    a = rng.integers(lo, hi, (n, n), dtype=np.int64)
    a = np.triu(a)
    a = a + np.triu(a, 1).T
    if not diag:
        np.fill_diagonal(a, 0)
    return a


# ----------------------------------------------------------------- host logic (CPU)


def test_primes_are_prime_and_descending():
    ps = exact._PRIMES
    assert ps[0] == 2147483647 and ps[1] == 2147483629 and ps[2] == 2147483587
    assert all(a > b for a, b in zip(ps, ps[1:]))
    for p in ps[:8]:
        assert all(p % q for q in range(3, 2000, 2))
    assert exact.primes_below(100, 5) == [97, 89, 83, 79, 73]


def test_crt_centred_lift_round_trips():
    ps = exact._PRIMES[:4]
    M = 1
    for p in ps:
        M *= p
    rng = np.random.default_rng(0)
    for x in [0, 1, -1, CFG3_EXACT, -CFG3_EXACT, M // 2, -(M // 2)] + [
        int(v) * 10**20 + int(w) for v, w in rng.integers(-10**9, 10**9, (20, 2))
    ]:
        assert exact._crt([x % p for p in ps], ps) == x


def test_bound_dominates_exact_values():
    for n in (2, 4, 6, 8, 10):
        for seed in range(3):
            a = _rand_int_sym(n, seed)
            rows = a.tolist()
            assert abs(hafnian_exact_dp(np.where(np.eye(n, dtype=bool), 0, a))) <= exact.hafnian_bound(
                [[0 if i == j else rows[i][j] for j in range(n)] for i in range(n)], False)
            assert abs(hafnian_exact_dp(a, loops=True)) <= exact.hafnian_bound(rows, True)


def test_prime_count_covers_bound():
    # cfg3 (0/1, n=40): (39)!! < 2^79 -> three 31-bit primes suffice, as in SURVEY.md
    rows = exact._as_int_matrix(workloads.cfg3())
    b = exact.hafnian_bound(rows, False)
    assert b == double_factorial(39)
    assert exact._PRIMES[0] * exact._PRIMES[1] * exact._PRIMES[2] > 2 * b


def test_exact_input_semantics():
    with pytest.raises(AsymmetricInput):
        exact._as_int_matrix([[0, 1], [2, 0]])
    with pytest.raises(NonSquare):
        exact._as_int_matrix([[0, 1, 2], [1, 0, 3]])
    with pytest.raises(ValueError):
        exact._as_int_matrix([[0, 0.5], [0.5, 0]])
    with pytest.raises(ValueError):
        exact._as_int_matrix([[0, 1j], [1j, 0]])
    assert exact._as_int_matrix(np.array([[0, 2.0], [2.0, 0]], dtype=complex)) == [[0, 2], [2, 0]]
    big = 10**30
    assert exact._as_int_matrix([[0, big], [big, 0]]) == [[0, big], [big, 0]]
    # shape errors raised before any device work
    with pytest.raises(OddDimension):
        exact.hafnian_exact(np.zeros((3, 3), int))
    with pytest.raises(TooLarge):
        exact.hafnian_exact(np.zeros((66, 66), int))
    assert exact.hafnian_exact(np.zeros((0, 0), int)) == 1


def test_contiguous_shards_partition_the_masks():
    for D in (4, 10, 20, 26):
        for k in (1, 2, 3, 8):
            sh = exact._contiguous_shards(D, k)
            assert sh[0][0] == 1 and sh[-1][1] == 1 << D
            assert all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
            assert len(sh) <= k


def test_exact_dp_oracle_closed_forms():
    for n in (2, 4, 6, 8, 10, 12):
        assert hafnian_exact_dp(np.ones((n, n), int)) == double_factorial(n - 1)
        assert hafnian_exact_dp(np.ones((n, n), int), loops=True) == telephone(n)


# ----------------------------------------------------------------- device (GPU)

gpu = pytest.mark.gpu


@gpu
def test_exact_random_integer_matrices_vs_dp():
    for n in range(2, 17, 2):
        for seed in range(3):
            a = _rand_int_sym(n, 100 * n + seed)
            assert exact.hafnian_exact(a) == hafnian_exact_dp(np.where(np.eye(n, dtype=bool), 0, a)), (n, seed)
            assert exact.loop_hafnian_exact(a) == hafnian_exact_dp(a, loops=True), (n, seed)


@gpu
def test_exact_large_entries_beyond_float_range():
    """Entries ~2^40: the hafnian is far beyond 2^64 and 2^53; exact equality holds."""
    rng = np.random.default_rng(7)
    for n in (8, 12, 14):
        a = [[0] * n for _ in range(n)]
        for i in range(n):
            for j in range(i, n):
                v = int(rng.integers(-(1 << 40), 1 << 40))
                a[i][j] = a[j][i] = v
        want = hafnian_exact_dp([[0 if i == j else a[i][j] for j in range(n)] for i in range(n)])
        assert abs(want) > 1 << 64
        assert exact.hafnian_exact(a) == want
        assert exact.loop_hafnian_exact(a) == hafnian_exact_dp(a, loops=True)


@gpu
def test_exact_complete_graphs_and_telephone():
    for n in (2, 10, 20, 30, 40):
        assert exact.hafnian_exact(np.ones((n, n), int)) == double_factorial(n - 1), n
    for n in (2, 10, 20, 30):
        assert exact.loop_hafnian_exact(np.ones((n, n), int)) == telephone(n), n


@gpu
def test_exact_bipartite_equals_permanent():
    rng = np.random.default_rng(3)
    for k in (3, 5, 7):
        W = rng.integers(-4, 5, (k, k))
        # Ryser in exact ints
        perm = 0
        for s in range(1, 1 << k):
            cols = [j for j in range(k) if s >> j & 1]
            prod = 1
            for i in range(k):
                prod *= sum(int(W[i, j]) for j in cols)
            perm += (-1) ** len(cols) * prod
        perm *= (-1) ** k
        B = bipartite_embedding(W).real.astype(np.int64)
        assert exact.hafnian_exact(B) == perm


@gpu
def test_exact_cfg3_known_answer():
    """the ER(0.5) n=40 perfect-matching count."""
    assert exact.hafnian_exact(workloads.cfg3()) == CFG3_EXACT


@gpu
def test_exact_more_primes_same_answer():
    a = _rand_int_sym(16, 5)
    base = exact.hafnian_exact(a)
    assert exact.hafnian_exact(a, n_primes=6) == base


@gpu
def test_modp_residues_shard_additively():
    """Any split of the mask interval sums to the same residues (the multi-device
    plan is exact, independent of the partition)."""
    n = 24
    a = _rand_int_sym(n, 11, diag=False)
    rows = a.tolist()
    primes = exact._PRIMES[:3]
    perm = [i ^ 1 for i in range(n)]
    at = np.array([[[rows[perm[i]][j] % p for j in range(n)] for i in range(n)] for p in primes], np.uint32)
    dg = np.zeros((3, n), np.uint32)
    full, _ = kernels.modp_sums(at, dg, primes, n // 2, 1, 1 << (n // 2), False)
    for k in (2, 3, 5):
        acc = np.zeros(3, object)
        for lo, hi in exact._contiguous_shards(n // 2, k):
            r, _ = kernels.modp_sums(at, dg, primes, n // 2, lo, hi, False)
            acc += r.astype(object)
        assert [int(x) % p for x, p in zip(acc, primes)] == [int(x) for x in full]
    want = hafnian_exact_dp(a) if n <= 20 else None
    got = exact._crt([int(x) for x in full], primes)
    assert got == exact.hafnian_exact(a)
    if want is not None:
        assert got == want


@gpu
def test_exact_matches_float_engine_where_float_is_exact():
    from paper_1805_12498_b200 import engine

    for n in (10, 16, 20):
        a = _rand_int_sym(n, n, lo=-2, hi=3)
        f = engine.hafnian(a.astype(np.complex128))
        e = exact.hafnian_exact(a)
        assert abs(f.real - e) <= 1e-6 * max(1, abs(e)) and abs(f.imag) < 1e-6 * max(1, abs(e))


def test_exact_no_cpu_fallback(monkeypatch):
    if has_gpu():
        pytest.skip("device present")
    from paper_1805_12498_b200.errors import DeviceError

    with pytest.raises(DeviceError):
        exact.hafnian_exact(np.ones((4, 4), int))


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_modp_at_n64_matches_float_partial():
    """D = 32 (n = 64, the 32-bit-mask limit) in GF(p): the signed sum over masks [1, 2^12)
    of a 0/1 matrix, lifted by CRT from five primes (product ~2^155), must agree with the
    bit-exact MIRROR float partial (== the reference) to float rounding (|sum| ~ 5e32; a
    wrong residue would lift to an unrelated ~1e46 integer)."""
    rng = np.random.default_rng(640)
    adj = np.triu((rng.uniform(size=(64, 64)) < 0.5).astype(np.int64), 1)
    A = adj + adj.T
    from paper_1805_12498_b200 import engine

    at, dg, nh = engine._prepare(A.astype(complex), False)
    sums, fails = kernels.sum_mask_range(at, dg, nh, 1, 1 << 12, 1, 1, False, arith="mirror")
    want = complex(sums[0])
    assert not fails.any() and abs(want) > 1e30
    primes = exact._PRIMES[:5]
    perm = [i ^ 1 for i in range(64)]
    atp = np.array([[[int(A[perm[i], j]) % p for j in range(64)] for i in range(64)] for p in primes],
                   np.uint32)
    dgp = np.zeros((len(primes), 64), np.uint32)
    res, _ = kernels.modp_sums(atp, dgp, primes, 32, 1, 1 << 12, False)
    got = exact._crt([int(r) for r in res], list(primes))
    assert abs(got - want.real) <= 1e-10 * abs(want.real) and abs(want.imag) <= 1e-10 * abs(want)
