"""Host-side logic that needs no GPU: cost model and shard planner, option and
input validation, the reduction contract, workloads, and the no-fallback rule."""

import math

import numpy as np
import pytest

from paper_1805_12498_b200 import costmodel, engine, workloads
from paper_1805_12498_b200.errors import AsymmetricInput, NonSquare, OddDimension, TooLarge
from paper_1805_12498_b200.matrix import PairSubset, pair_swap, validate_or_symmetrize


def test_flop_totals_match_survey():
    # SURVEY.md 8(d) table
    assert costmodel.flops_total(10) == 9_886_360
    assert costmodel.flops_total(12) == 66_332_400
    assert costmodel.flops_total(16, loops=True) == 4_695_110_400
    assert costmodel.flops_total(20) == 73_938_187_600
    assert abs(costmodel.flops_total(26) / 1.0172e13 - 1) < 1e-4
    assert abs(costmodel.flops_of_range(0, 1 << 20, 26) / 7.6095e10 - 1) < 1e-4


def test_count_below_brute_force():
    D = 10
    pc = [bin(x).count("1") for x in range(1 << D)]
    for x in (0, 1, 5, 17, 300, 511, 1023, 1024):
        for p in range(D + 1):
            assert costmodel.count_below(x, p, D) == sum(1 for y in range(x) if pc[y] == p)


def test_range_bounds_match_reference_partition():
    for nh, nr in ((10, 512), (5, 31), (12, 512)):
        total = 1 << nh
        w = -(-(total - 1) // nr)
        for r, (a, b) in enumerate(costmodel.range_bounds(nh, nr)):
            assert a == min(1 + r * w, total) and b == min(a + w, total)


def test_lpt_balances_better_than_round_robin():
    costs = costmodel.range_costs(26, 512)
    for k in (2, 4, 8):
        lpt = costmodel.imbalance(costs, costmodel.lpt_shards(costs, k))
        rr = costmodel.imbalance(costs, [list(range(w, 512, k)) for w in range(k)])
        assert lpt < 1.005 < rr
    sh = costmodel.lpt_shards(costs, 8)
    assert sorted(i for s in sh for i in s) == list(range(512))


def test_options_validation():
    with pytest.raises(ValueError):
        engine.EngineOptions(backend="magic").validate()
    with pytest.raises(ValueError):
        engine.EngineOptions(reduction="sloppy").validate()
    with pytest.raises(ValueError):
        engine.EngineOptions(threads=0).validate()
    with pytest.raises(ValueError):
        engine.EngineOptions(arith="sloppy").validate()
    with pytest.raises(ValueError):
        engine.EngineOptions(devices=0).validate()


def test_env_threads(monkeypatch):
    monkeypatch.setenv("HAFNIUM_THREADS", "3")
    assert engine.EngineOptions().resolved_threads() == 3


def test_input_semantics():
    with pytest.raises(NonSquare):
        validate_or_symmetrize(np.zeros((2, 3)))
    a = np.array([[0, 1], [1.5, 0]], complex)
    with pytest.raises(AsymmetricInput):
        validate_or_symmetrize(a)
    b = np.array([[0, 1], [1 + 1e-14, 0]], complex)
    m = validate_or_symmetrize(b)
    assert m.entries[1, 0] == m.entries[0, 1] == 1  # upper mirrored onto lower
    with pytest.raises(OddDimension):
        engine._prepare(np.zeros((3, 3)), False)
    with pytest.raises(TooLarge):
        engine._prepare(np.zeros((66, 66)), False)
    assert engine._prepare(np.zeros((64, 64)), False)[2] == 32  # n = 64: D = 32 (32-bit masks)
    x = np.arange(16).reshape(4, 4).astype(complex)
    assert np.array_equal(pair_swap(x), x[[1, 0, 3, 2]])
    assert PairSubset(0b101, 3).vertex_indices().tolist() == [0, 1, 4, 5]


def test_prepare_zeroes_diagonal_only_for_hafnian():
    a = workloads.cfg2(n=6)
    at, dg, nh = engine._prepare(a, False)
    assert nh == 3 and not dg.any()
    at2, dg2, _ = engine._prepare(a, True)
    assert np.array_equal(dg2, np.diag(a))


def test_tree_reduce_shape():
    assert engine.tree_reduce([1, 2, 3]) == 6
    assert engine.tree_reduce([]) == 0


def test_tree_reduce_matches_reference_list_form_bitwise():
    """The array form adds the same pairs in the same association as the reference's list
    form (engine.py:87-97), for every length (odd tails carried up) and non-finite values."""
    def ref(values):
        vals = [complex(v) for v in values]
        if not vals:
            return 0.0 + 0.0j
        while len(vals) > 1:
            nxt = [vals[i] + vals[i + 1] for i in range(0, len(vals) - 1, 2)]
            if len(vals) % 2:
                nxt.append(vals[-1])
            vals = nxt
        return vals[0]

    rng = np.random.default_rng(11)
    for n in list(range(0, 20)) + [31, 33, 511, 512, 513, 1000]:
        v = (rng.normal(size=n) + 1j * rng.normal(size=n)) * 10.0 ** rng.integers(-9, 9, size=n)
        a, b = engine.tree_reduce(v), ref(v)
        assert np.array([a]).view(np.uint64).tolist() == np.array([b]).view(np.uint64).tolist(), n
        assert engine.tree_reduce(list(v)) == b
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        bad = engine.tree_reduce(np.array([np.inf, -np.inf, 1.0, 2.0 + 0j]))
    assert np.isnan(bad.real) and bad.imag == 0.0


def test_workload_generators():
    a3 = workloads.cfg3()
    assert a3.shape == (40, 40) and np.count_nonzero(np.triu(a3.real, 1)) == 393
    a1 = workloads.cfg1(0)
    assert a1.shape == (24, 24) and np.abs(a1 - a1.T).max() < 1e-12
    assert workloads.cfg4(3, 52).shape == (52, 52)


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_1805_12498_b200.errors import DeviceError

    with pytest.raises(DeviceError):
        engine.hafnian(workloads.cfg0(n=4))


def test_multi_device_plans_with_mocked_devices(monkeypatch):
    """hafnian(..., devices=N) host logic with the per-device range-list call replaced
    by the CPU oracle: the deterministic path reassembles the partials in range order
    (bit-identical to the single-device oracle result for every N); the fast path sums
    per device and agrees to rounding."""
    from oracle import oracle as O
    from paper_1805_12498_b200 import kernels

    def fake_range_list(atilde, diag, n_half, n_ranges, ranges, backend, loops, cap=30, *,
                        arith=None, device=None):
        total = 1 << n_half
        width = -(-(total - 1) // n_ranges)
        sums, fails = [], []
        for r in ranges:
            a = min(1 + int(r) * width, total)
            b = min(a + width, total)
            s, f = O.sum_mask_range(atilde, diag, n_half, a, b, 1, backend, loops, cap)
            sums.append(s[0])
            fails.append(f[0])
        return np.array(sums, np.complex128), np.array(fails, np.int64)

    monkeypatch.setattr(kernels, "sum_range_list", fake_range_list)
    monkeypatch.setattr(kernels, "device_count", lambda: 8)
    O.build()
    A = workloads.cfg0()
    want, _ = O.hafnian(A, backend=1)
    for n_dev in (1, 2, 3, 8):
        if n_dev == 1:
            continue  # the single-device path calls sum_subsets_det, not the mock
        got = engine.hafnian(A, backend="charpoly", devices=n_dev)
        assert got == want, n_dev
        fast = engine.hafnian(A, backend="charpoly", devices=n_dev, reduction="fast")
        assert abs(fast - want) <= 1e-12 * abs(want), n_dev
    lw, _ = O.hafnian(workloads.cfg2(n=12), backend=1, include_loops=True)
    assert engine.loop_hafnian(workloads.cfg2(n=12), backend="charpoly", devices=3) == lw


def test_more_devices_than_visible_is_a_clear_error(monkeypatch):
    """devices > visible CUDA devices raises DeviceError up front (no hang, no partial run)."""
    from paper_1805_12498_b200 import kernels
    from paper_1805_12498_b200.errors import DeviceError

    monkeypatch.setattr(kernels, "device_count", lambda: 2)
    with pytest.raises(DeviceError, match="devices=4"):
        engine.hafnian(workloads.cfg0(), backend="charpoly", devices=4)


def test_arith_backend_combinations_validate():
    for backend in ("spectral", "charpoly"):
        for arith in ("fast", "mirror"):
            engine.EngineOptions(backend=backend, arith=arith).validate()
    with pytest.raises(ValueError, match="arith"):
        engine.EngineOptions(arith="exact").validate()
