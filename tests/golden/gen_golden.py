"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run here (the container that has /root/reference), never on the GPU box:

    NUMBA_CACHE_DIR=/tmp/nc python tests/golden/gen_golden.py

It imports the unmodified reference package (hafnium 0.1.0, numba kernels)
from /root/reference/pkg/src and records, for the canonical workloads of
SURVEY.md Appendix A plus small random cases:

* terms.npz      per-term values ``_numba.subset_term`` (both backends, with
                 and without loops) for masks sampled across every popcount;
* ranges.npz     the 512 per-range Kahan partials of ``_numba.sum_subsets_det``
                 and the public ``hafnium.hafnian / loop_hafnian`` results;
* range_n52.npz  masks [0, 2^20) of the n=52 / n=56 inputs, 512 equal chunks,
                 Kahan per chunk, via a small njit harness around
                 ``_numba.subset_term`` (the reference has no range API;
                 SURVEY.md 8(c));
* powertraces.npz power traces / charpoly coefficients / exp coefficients of
                 random matrices through the reference kernel entry points.

Input matrices are stored in the fixtures, so consumers never regenerate
them (LAPACK-based cfg1 inputs could differ in the last ulp across CPUs).
"""

from __future__ import annotations

import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nc")
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import numba  # noqa: E402
import numpy as np  # noqa: E402

import hafnium  # noqa: E402
from hafnium.engine import _prepare, tree_reduce  # noqa: E402
from hafnium.kernels import _numba as nb  # noqa: E402

from paper_1805_12498_b200 import workloads as W  # noqa: E402

sys.path.insert(0, os.path.dirname(HERE))
from conftest import digest  # noqa: E402

THREADS = os.cpu_count()


def sample_masks(n_half: int, per_popcount: int, seed: int) -> np.ndarray:
    """Up to ``per_popcount`` masks of every popcount 1..n_half (plus the full mask)."""
    rng = np.random.default_rng(seed)
    out = []
    for m in range(1, n_half + 1):
        for _ in range(per_popcount):
            bits = rng.choice(n_half, size=m, replace=False)
            out.append(int(np.sum(np.left_shift(np.uint64(1), bits.astype(np.uint64)))))
    out.append((1 << n_half) - 1)
    out.append(1)
    return np.unique(np.array(out, dtype=np.uint64))


def ref_terms(atilde, diag, n_half, masks, backend, loops):
    vals = np.zeros(len(masks), np.complex128)
    st = np.zeros(len(masks), np.int64)
    for q, m in enumerate(masks):
        t, s = nb.subset_term(atilde, diag, int(m), n_half, backend, loops, nb.SWEEP_CAP_MULT)
        vals[q] = t
        st[q] = s
    return vals, st


def random_sym(n, seed):
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
    return (a + a.T) / 2


def term_cases():
    cases = [
        ("cfg0", W.cfg0(), False, 24),
        ("cfg1s0", W.cfg1(0), False, 16),
        ("cfg2", W.cfg2(), True, 16),
        ("cfg2_haf", W.cfg2(), False, 8),
        ("cfg3", W.cfg3(), False, 12),
        ("cfg4_n52s3", W.cfg4(3, 52), False, 6),
        ("cfg4_n56s4", W.cfg4(4, 56), False, 3),
    ]
    for n in (2, 4, 6, 8, 10, 12, 14):
        cases.append((f"rand{n}", random_sym(n, 900 + n), False, 8))
        cases.append((f"rand{n}_loops", random_sym(n, 950 + n), True, 8))
    # structured: complete graph and all-ones with loops (exact ties in the pivot search)
    k = np.ones((16, 16), complex)
    np.fill_diagonal(k, 0)
    cases.append(("complete16", k, False, 8))
    cases.append(("ones12_loops", np.ones((12, 12), complex), True, 8))
    return cases


def gen_terms():
    out = {}
    for name, A, loops, per in term_cases():
        at, dg, nh = _prepare(A, loops)
        masks = sample_masks(nh, per, seed=len(name) * 7 + nh)
        out[f"{name}/A"] = np.asarray(A, np.complex128)
        out[f"{name}/loops"] = np.array(loops)
        out[f"{name}/masks"] = masks
        for backend in (1, 0):
            t0 = time.time()
            vals, st = ref_terms(at, dg, nh, masks, backend, loops)
            out[f"{name}/terms_b{backend}"] = vals
            out[f"{name}/status_b{backend}"] = st
            print(f"terms {name} b{backend}: {len(masks)} masks {time.time() - t0:.1f}s", flush=True)
    np.savez_compressed(os.path.join(HERE, "terms.npz"), **out)


def gen_ranges():
    out = {}
    cases = [("cfg0", W.cfg0(), False, (1, 0)), ("cfg2", W.cfg2(), True, (1, 0)),
             ("cfg3", W.cfg3(), False, (1, 0))]
    for s in range(4):
        cases.append((f"cfg1s{s}", W.cfg1(s), False, (1, 0)))
    for n in (2, 4, 6, 8, 10, 12):
        cases.append((f"rand{n}", random_sym(n, 300 + n), False, (1, 0)))
        cases.append((f"rand{n}_loops", random_sym(n, 400 + n), True, (1, 0)))
    for name, A, loops, backends in cases:
        at, dg, nh = _prepare(A, loops)
        nr = min((1 << nh) - 1, 512)
        out[f"{name}/A"] = np.asarray(A, np.complex128)
        out[f"{name}/loops"] = np.array(loops)
        for backend in backends:
            t0 = time.time()
            sums, fails = nb.sum_subsets_det(at, dg, nh, backend, loops, THREADS, nr,
                                             nb.SWEEP_CAP_MULT)
            bname = "charpoly" if backend == 1 else "spectral"
            f = hafnium.loop_hafnian if loops else hafnium.hafnian
            res = f(A, backend=bname, threads=THREADS)
            assert res == tree_reduce(sums)
            fsums, ffails = nb.sum_subsets_fast(at, dg, nh, backend, loops, 3, nr,
                                                nb.SWEEP_CAP_MULT)
            out[f"{name}/partials_b{backend}"] = sums
            out[f"{name}/fails_b{backend}"] = fails
            out[f"{name}/result_b{backend}"] = np.array(res)
            out[f"{name}/fast3_b{backend}"] = fsums
            print(f"ranges {name} b{backend}: {res} {time.time() - t0:.1f}s", flush=True)
    np.savez_compressed(os.path.join(HERE, "ranges.npz"), **out)


@numba.njit(parallel=True)
def _range_driver(atilde, diag, n_half, lo, hi, n_chunks, backend, loops, cap):
    """SURVEY 8(c) harness: Kahan per chunk over masks [lo, hi), mask 0 skipped."""
    width = (hi - lo + n_chunks - 1) // n_chunks
    sums = np.zeros(n_chunks, np.complex128)
    fails = np.zeros(n_chunks, np.int64)
    for r in numba.prange(n_chunks):
        a = lo + r * width
        b = min(a + width, hi)
        s = 0.0 + 0.0j
        comp = 0.0 + 0.0j
        for mask in range(a, b):
            if mask == 0:
                continue
            term, st = nb.subset_term(atilde, diag, mask, n_half, backend, loops, cap)
            if st != 0:
                fails[r] = st
            y = term - comp
            t = s + y
            comp = (t - s) - y
            s = t
        sums[r] = s
    return sums, fails


def gen_range_n52():
    out = {}
    for name, A, backends in [("n52s3", W.cfg4(3, 52), (1, 0)), ("n52s4", W.cfg4(4, 52), (1,)),
                              ("n56s4", W.cfg4(4, 56), (1,))]:
        at, dg, nh = _prepare(A, False)
        out[f"{name}/A"] = A
        for backend in backends:
            t0 = time.time()
            sums, fails = _range_driver(at, dg, nh, 0, 1 << 20, 512, backend, False,
                                        nb.SWEEP_CAP_MULT)
            out[f"{name}/partials_b{backend}"] = sums
            out[f"{name}/fails_b{backend}"] = fails
            out[f"{name}/result_b{backend}"] = np.array(tree_reduce(sums))
            print(f"range {name} b{backend}: {tree_reduce(sums)} {time.time() - t0:.1f}s", flush=True)
    np.savez_compressed(os.path.join(HERE, "range_n52.npz"), **out)


def gen_batch(count: int = 4096):
    """cfg1: the full 4096-matrix batch through the reference's public API, looped as
    the reference itself has to (no batch API; SURVEY.md finding 6), both backends."""
    out = {"seeds": np.arange(count, dtype=np.int64)}
    mats = [W.cfg1(s) for s in range(count)]
    out["digests"] = np.array([digest(a) for a in mats], dtype=np.uint64)
    for backend, bname in ((1, "charpoly"), (0, "spectral")):
        t0 = time.time()
        res = np.array([hafnium.hafnian(a, backend=bname, threads=THREADS) for a in mats])
        out[f"result_b{backend}"] = res
        out[f"seconds_b{backend}"] = np.array(time.time() - t0)
        print(f"batch cfg1 x{count} {bname}: {time.time() - t0:.1f}s", flush=True)
    np.savez_compressed(os.path.join(HERE, "batch_cfg1.npz"), **out)


def gen_range_n64():
    """n = 64 (D = 32, the device's 32-bit-mask limit): the identical range [0, 2^20) and
    per-term values for sampled masks of the large classes (S = 42..64)."""
    out = {}
    A = W.cfg4(5, 64)
    at, dg, nh = _prepare(A, False)
    out["n64s5/A"] = A
    t0 = time.time()
    sums, fails = _range_driver(at, dg, nh, 0, 1 << 20, 512, 1, False, nb.SWEEP_CAP_MULT)
    out["n64s5/partials_b1"] = sums
    out["n64s5/fails_b1"] = fails
    out["n64s5/result_b1"] = np.array(tree_reduce(sums))
    rng = np.random.default_rng(64)
    masks = []
    for m in (21, 24, 27, 30, 31, 32):
        for _ in range(3 if m < 32 else 1):
            bits = rng.choice(nh, size=m, replace=False)
            masks.append(int(np.sum(np.left_shift(np.uint64(1), bits.astype(np.uint64)))))
    masks = np.array(sorted(set(masks)), dtype=np.uint64)
    vals, st = ref_terms(at, dg, nh, masks, 1, False)
    out["n64s5/masks"] = masks
    out["n64s5/terms_b1"] = vals
    out["n64s5/status_b1"] = st
    print(f"range n64s5: {tree_reduce(sums)} {time.time() - t0:.1f}s", flush=True)
    np.savez_compressed(os.path.join(HERE, "range_n64.npz"), **out)


def gen_powertraces():
    out = {}
    rng = np.random.default_rng(2024)
    for q in range(60):
        m = int(rng.integers(1, 21))
        K = int(rng.integers(1, 30))
        b = rng.uniform(-1, 1, (m, m)) + 1j * rng.uniform(-1, 1, (m, m))
        out[f"{q}/b"] = b
        out[f"{q}/K"] = np.array(K)
        t, ok = nb.power_traces_charpoly(b.copy(), K)
        out[f"{q}/charpoly_traces"] = t
        out[f"{q}/charpoly_ok"] = np.array(ok)
        out[f"{q}/coeffs"] = nb.charpoly_coefficients(b.copy())
        ts, sweeps, conv = nb.power_traces_spectral(b.copy(), K, nb.SWEEP_CAP_MULT)
        out[f"{q}/spectral_traces"] = ts
        out[f"{q}/spectral_sweeps"] = np.array(sweeps)
        out[f"{q}/spectral_conv"] = np.array(conv)
        D = int(rng.integers(1, 30))
        s = np.concatenate([[0], rng.normal(size=D) + 1j * rng.normal(size=D)])
        out[f"{q}/series"] = s
        out[f"{q}/exp_top"] = np.array(nb._exp_top(s))
    np.savez_compressed(os.path.join(HERE, "powertraces.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["terms", "ranges", "range_n52", "powertraces"]
    print("numba", numba.__version__, "numpy", np.__version__, "threads", THREADS)
    if "powertraces" in which:
        gen_powertraces()
    if "terms" in which:
        gen_terms()
    if "ranges" in which:
        gen_ranges()
    if "range_n52" in which:
        gen_range_n52()
    if "batch" in which:
        gen_batch()
    if "range_n64" in which:
        gen_range_n64()
