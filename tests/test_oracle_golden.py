"""Pin the C oracle (oracle/hafnian_oracle.c) to the reference itself.

The fixtures were produced by running the unmodified reference (numba kernels)
in tests/golden/gen_golden.py.  The oracle restates the reference's operation
sequence exactly, so every comparison here is BIT-EXACT.  CPU only.
"""

import numpy as np
import pytest

from conftest import bits, load_golden
from oracle import oracle as O


def _prep(A, loops):
    return O.prepare(A, loops)


def test_terms_bit_exact_all_cases():
    g = load_golden("terms.npz")
    checked = 0
    for name, case in g.items():
        loops = bool(case["loops"])
        at, dg, nh = _prep(case["A"], loops)
        for backend in (1, 0):
            vals, st = O.terms(at, dg, nh, case["masks"], backend, loops)
            assert np.array_equal(st, case[f"status_b{backend}"]), name
            same = bits(vals) == bits(case[f"terms_b{backend}"])
            assert same.all(), f"{name} backend {backend}: {np.count_nonzero(~same)} words differ"
            checked += vals.size
    assert checked > 2000


def test_range_partials_and_results_bit_exact():
    g = load_golden("ranges.npz")
    for name, case in g.items():
        loops = bool(case["loops"])
        at, dg, nh = _prep(case["A"], loops)
        nr = min((1 << nh) - 1, 512)
        for backend in (1, 0):
            key = f"partials_b{backend}"
            if key not in case:
                continue
            if name == "cfg3" and backend == 0:
                continue  # 40+ s of CPU; covered by the charpoly backend and the GPU tests
            sums, fails = O.sum_subsets_det(at, dg, nh, backend, loops, 8, nr)
            assert (bits(sums) == bits(case[key])).all(), f"{name} b{backend}"
            assert np.array_equal(fails, case[f"fails_b{backend}"])
            assert O.tree_reduce(sums) == complex(case[f"result_b{backend}"])
            fs, _ = O.sum_subsets_fast(at, dg, nh, backend, loops, 3, nr)
            assert (bits(fs) == bits(case[f"fast3_b{backend}"])).all(), f"{name} fast b{backend}"


def test_powertraces_bit_exact():
    g = load_golden("powertraces.npz")
    for q, case in g.items():
        b, K = case["b"], int(case["K"])
        t, ok = O.power_traces_charpoly(b, K)
        assert ok == bool(case["charpoly_ok"])
        assert (bits(t) == bits(case["charpoly_traces"])).all(), q
        assert (bits(O.charpoly_coefficients(b)) == bits(case["coeffs"])).all(), q
        ts, sweeps, conv = O.power_traces_spectral(b, K)
        assert conv == bool(case["spectral_conv"])
        assert sweeps == int(case["spectral_sweeps"])
        assert (bits(ts) == bits(case["spectral_traces"])).all(), q
        assert O.exp_top(case["series"]) == complex(case["exp_top"])


@pytest.mark.slow
def test_n52_range_bit_exact():
    g = load_golden("range_n52.npz")
    case = g["n52s3"]
    at, dg, nh = _prep(case["A"], False)
    sums, fails = O.sum_mask_range(at, dg, nh, 0, 1 << 20, 512, backend=1)
    assert (bits(sums) == bits(case["partials_b1"])).all()
    assert O.tree_reduce(sums) == complex(case["result_b1"])


def test_appendix_a_values():
    """SURVEY.md Appendix A reference values (charpoly and spectral, cfg0)."""
    from paper_1805_12498_b200 import workloads as W

    assert O.hafnian(W.cfg0(), 1)[0] == (-633.6415330499929 + 14.539502055681396j)
    assert O.hafnian(W.cfg0(), 0)[0] == (-633.641533051311 + 14.539502051755335j)
