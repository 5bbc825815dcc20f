"""The reference itself, running on the GPU through its own plugin API.

The unmodified reference package (hafnium 0.1.0, installed in baseline/_ref by the
recipe in DESIGN.md) is imported and its kernel selector is pointed at
paper_1805_12498_b200.refplugin -- what INTEGRATION.md's ``_b200`` module plus
``HAFNIUM_KERNELS=b200`` does.  The reference's own engine (``hafnium.hafnian``,
``loop_hafnian``, ``subset_term``, its option handling, tree reduction and error
mapping) then drives the device kernels, and the hot-path known-answer tests of
pkg/tests/test_engine.py:46-176 / :311-320 (restated here) run through
it.  In MIRROR arithmetic every result must also be bit-identical to the same call
on the reference's own numba kernels.
"""

import math
import os
import sys

import numpy as np
import pytest

from conftest import REPO, has_gpu, random_symmetric

REF = os.path.join(REPO, "baseline", "_ref")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device"),
              pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "hafnium")),
                                 reason="reference not installed in baseline/_ref")]


@pytest.fixture(scope="module")
def hafnium():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/hafb_numba_cache")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import hafnium as h

    return h


@pytest.fixture
def on_b200(hafnium, monkeypatch):
    """Select the B200 plugin behind the reference's kernel selector."""
    from paper_1805_12498_b200 import refplugin

    monkeypatch.setattr(hafnium.kernels, "active", lambda: refplugin)
    return refplugin


def test_selector_reaches_the_device(hafnium, on_b200, monkeypatch):
    from paper_1805_12498_b200 import _lib

    calls = []
    real = on_b200.sum_subsets_det
    monkeypatch.setattr(on_b200, "sum_subsets_det", lambda *a: calls.append(1) or real(*a))
    lib = _lib.load(require_device=True)
    lib.hafb_launch_count(1)
    hafnium.hafnian(random_symmetric(8, 1))
    assert calls and lib.hafb_launch_count(1) > 0


def test_empty_odd_single_pair_and_4x4(hafnium, on_b200):
    assert hafnium.hafnian(np.zeros((0, 0))) == 1
    with pytest.raises(hafnium.errors.OddDimension):
        hafnium.hafnian(np.ones((3, 3)))
    a = 0.3 - 1.7j
    assert abs(hafnium.hafnian(np.array([[0, a], [a, 0]])) - a) <= 1e-14 * abs(a)
    A = random_symmetric(4, 2)
    three = A[0, 1] * A[2, 3] + A[0, 2] * A[1, 3] + A[0, 3] * A[1, 2]
    assert abs(hafnium.hafnian(A) - three) <= 1e-12 * abs(three)


@pytest.mark.parametrize("backend", ["spectral", "charpoly"])
def test_diagonal_ignored_bitwise(hafnium, on_b200, backend):
    A = random_symmetric(10, 3)
    B = A.copy()
    np.fill_diagonal(B, 5.0 + 2.0j)
    assert hafnium.hafnian(A, backend=backend) == hafnium.hafnian(B, backend=backend)


@pytest.mark.parametrize("backend", ["spectral", "charpoly"])
def test_complete_graph_k20(hafnium, on_b200, backend):
    K = np.ones((20, 20), complex)
    np.fill_diagonal(K, 0)
    got = hafnium.hafnian(K, backend=backend)
    assert abs(got - 654729075) <= 1e-9 * 654729075  # 19!!


@pytest.mark.parametrize("m", [2, 3, 4, 5])
def test_bipartite_embedding_is_ryser_permanent(hafnium, on_b200, m):
    rng = np.random.default_rng(70 + m)
    W = rng.uniform(-1, 1, (m, m)) + 1j * rng.uniform(-1, 1, (m, m))
    per = hafnium.oracle.permanent_ryser(W)
    assert abs(hafnium.hafnian(hafnium.oracle.bipartite_embedding(W)) - per) <= 1e-9 * max(1, abs(per))


@pytest.mark.parametrize("n", [2, 4, 6, 8, 10])
def test_random_vs_bruteforce_hafnian_and_loop(hafnium, on_b200, n):
    A = random_symmetric(n, n + 300)
    ref = hafnium.oracle.hafnian_bruteforce(A)
    assert abs(hafnium.hafnian(A) - ref) <= 1e-10 * max(1, abs(ref))
    L = random_symmetric(n, n + 400)
    lref = hafnium.oracle.loop_hafnian_bruteforce(L)
    assert abs(hafnium.loop_hafnian(L) - lref) <= 1e-10 * max(1, abs(lref))


def test_backends_agree_n12(hafnium, on_b200):
    A = random_symmetric(12, 17)
    s, c = hafnium.hafnian(A, backend="spectral"), hafnium.hafnian(A, backend="charpoly")
    assert abs(s - c) <= 1e-8 * abs(c)


def test_loop_hafnian_kats(hafnium, on_b200):
    assert abs(hafnium.loop_hafnian(np.ones((10, 10))) - 9496) <= 1e-9 * 9496  # T(10)
    d = np.array([0.5 + 1j, -2.0, 3.0 - 0.5j, 1.5j])
    want = np.prod(d)
    assert abs(hafnium.loop_hafnian(np.diag(d)) - want) <= 1e-12 * abs(want)
    A = random_symmetric(8, 5)
    np.fill_diagonal(A, 0)
    assert hafnium.loop_hafnian(A) == hafnium.hafnian(A)  # zero diagonal: bitwise


@pytest.mark.parametrize("mu", [0.5, 2.0, 3 + 4j])
def test_homogeneity(hafnium, on_b200, mu):
    A = random_symmetric(10, 21)
    h = hafnium.hafnian(A)
    assert abs(hafnium.hafnian(mu * A) - mu ** 5 * h) <= 1e-10 * abs(mu ** 5 * h)


def test_subset_terms(hafnium, on_b200):
    K4 = np.ones((4, 4), complex)
    np.fill_diagonal(K4, 0)
    total = sum(hafnium.subset_term(K4, m) for m in (1, 2, 3))
    assert abs(total - 3) <= 1e-12
    A = random_symmetric(8, 9)
    s = sum(hafnium.subset_term(A, m) for m in range(1, 16))
    ref = hafnium.oracle.hafnian_bruteforce(A)
    assert abs(s - ref) <= 1e-10 * max(1, abs(ref))
    with pytest.raises(ValueError):
        hafnium.subset_term(A, 0)
    with pytest.raises(ValueError):
        hafnium.subset_term(A, 16)


def test_sweep_cap_zero_propagates(hafnium, on_b200, monkeypatch):
    """The reference monkeypatches SWEEP_CAP_MULT on the ACTIVE module (test_engine.py:311-320)."""
    monkeypatch.setattr(on_b200, "SWEEP_CAP_MULT", 0)
    A = random_symmetric(8, 15)
    with pytest.raises(hafnium.errors.EigensolverNoConvergence):
        hafnium.hafnian(A, backend="spectral")


@pytest.mark.parametrize("n,loops,backend", [(12, False, "spectral"), (16, False, "charpoly"),
                                             (14, True, "charpoly"), (12, True, "spectral")])
def test_mirror_bit_identical_to_numba_kernels(hafnium, monkeypatch, n, loops, backend):
    """Same reference engine, two kernel modules: numba (CPU) and the B200 plugin (MIRROR),
    both reductions (the fast one deals ranges to 3 workers)."""
    from paper_1805_12498_b200 import refplugin

    monkeypatch.setenv("HAFB200_ARITH", "mirror")
    A = random_symmetric(n, 500 + n)
    f = hafnium.loop_hafnian if loops else hafnium.hafnian
    runs = [dict(backend=backend, threads=4), dict(backend=backend, threads=3, reduction="fast")]
    want = [f(A, **kw) for kw in runs]  # numba kernels (the reference default)
    monkeypatch.setattr(hafnium.kernels, "active", lambda: refplugin)
    got = [f(A, **kw) for kw in runs]
    assert got == want


def test_fast_arith_through_the_plugin(hafnium, on_b200, monkeypatch):
    """HAFB200_ARITH=fast reaches the FAST kernels through the reference's selector."""
    monkeypatch.setenv("HAFB200_ARITH", "fast")
    K = np.ones((16, 16), complex)
    np.fill_diagonal(K, 0)
    got = hafnium.hafnian(K, backend="charpoly")
    assert abs(got - math.prod(range(1, 16, 2))) <= 1e-10 * 2027025
    A = random_symmetric(14, 33)
    monkeypatch.setenv("HAFB200_ARITH", "mirror")
    m = hafnium.hafnian(A, backend="charpoly")
    monkeypatch.setenv("HAFB200_ARITH", "fast")
    fst = hafnium.hafnian(A, backend="charpoly")
    assert abs(fst - m) <= 1e-10 * abs(m)
