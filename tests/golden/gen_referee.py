"""Generate tests/golden/referee*.npz: extended-precision referee values.

Run here (build container; CPU only):

    python tests/golden/gen_referee.py [small] [batch] [ranges] [full]

For every BASELINE config the same subset sum is evaluated by oracle/referee.c
in x87 long double (64-bit significand; binary128 for the small cases as a
check of the long double referee itself), so the double-precision results of
the reference, MIRROR (bit-identical to the reference) and FAST can be scored
against a value ~2000x more precise than any of them.

* referee.npz          cfg0, cfg2 (loops), cfg3, cfg1 seeds 0..3: full results;
                       the n=52 / n=56 identical ranges [0, 2^20) (seeds 3, 4);
                       per-term referee values for the terms.npz masks;
                       n = 64 (range_n64.npz): the range and its large-class terms
* referee_batch.npz    the 4096-matrix cfg1 batch (per matrix; input digests as
                       in batch_cfg1.npz)
* referee_full52.npz   the FULL n=52 seed-3 hafnian (2^26-1 terms, ~1 h on 8 cores)

Inputs are taken from the fixtures that hold them (ranges.npz, range_n52.npz),
so the referee scores exactly the matrices the reference was run on.
"""

from __future__ import annotations

import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

from oracle import referee as R  # noqa: E402
from paper_1805_12498_b200 import engine, workloads as W  # noqa: E402


def _cases(path):
    g = np.load(os.path.join(HERE, path))
    names = sorted({k.split("/", 1)[0] for k in g.files if "/" in k})
    return {nm: {k.split("/", 1)[1]: g[k] for k in g.files if k.startswith(nm + "/")} for nm in names}


def _store(out, key, hi, lo, sa):
    out[f"{key}/hi"] = np.array(hi)
    out[f"{key}/lo"] = np.array(lo)
    out[f"{key}/abs_sum"] = np.array(sa)


def gen_small(out):
    rng_cases = _cases("ranges.npz")
    for name in ("cfg0", "cfg2", "cfg3", "cfg1s0", "cfg1s1", "cfg1s2", "cfg1s3"):
        c = rng_cases[name]
        loops = bool(c["loops"])
        at, dg, nh = engine._prepare(c["A"], loops)
        t0 = time.time()
        hi, lo, sa = R.sum_range(at, dg, nh, 1, 1 << nh, loops)
        _store(out, name, hi, lo, sa)
        msg = f"{name}: {hi} cond {sa / abs(hi):.2e} ({time.time() - t0:.1f}s)"
        if nh <= 16:  # binary128 check of the long double referee
            qhi, qlo, _ = R.sum_range(at, dg, nh, 1, 1 << nh, loops, quad=True)
            out[f"{name}/quad_hi"] = np.array(qhi)
            out[f"{name}/quad_lo"] = np.array(qlo)
            msg += f" ld-vs-quad {R.rel_err(hi + lo, qhi, qlo):.1e}"
        for b in (1, 0):
            msg += f" ref_b{b} err {R.rel_err(complex(c[f'result_b{b}']), hi, lo):.2e}"
        print(msg, flush=True)
    tc = _cases("terms.npz")
    for name, c in tc.items():
        loops = bool(c["loops"])
        at, dg, nh = engine._prepare(c["A"], loops)
        out[f"terms_{name}/values"] = R.terms(at, dg, nh, c["masks"], loops)


def gen_ranges(out):
    cases = dict(_cases("range_n52.npz"))
    if os.path.exists(os.path.join(HERE, "range_n64.npz")):
        n64 = _cases("range_n64.npz")
        cases.update(n64)
        for name, c in n64.items():  # per-term referee values of the large-class masks
            at, dg, nh = engine._prepare(c["A"], False)
            out[f"terms_{name}/values"] = R.terms(at, dg, nh, c["masks"], False)
    for name, c in cases.items():
        at, dg, nh = engine._prepare(c["A"], False)
        t0 = time.time()
        hi, lo, sa = R.sum_range(at, dg, nh, 0, 1 << 20, False)
        _store(out, f"range_{name}", hi, lo, sa)
        print(f"range {name}: {hi} cond {sa / abs(hi):.2e} ref_b1 err "
              f"{R.rel_err(complex(c['result_b1']), hi, lo):.2e} ({time.time() - t0:.1f}s)", flush=True)


def gen_batch():
    sys.path.insert(0, os.path.dirname(HERE))
    from conftest import digest

    count = 4096
    res_hi = np.zeros(count, np.complex128)
    res_lo = np.zeros(count, np.complex128)
    absum = np.zeros(count)
    dig = np.zeros(count, np.uint64)
    t0 = time.time()
    for s in range(count):
        A = W.cfg1(s)
        dig[s] = digest(A)
        at, dg, nh = engine._prepare(A, False)
        res_hi[s], res_lo[s], absum[s] = R.sum_range(at, dg, nh, 1, 1 << nh, False)
    print(f"batch referee x{count}: {time.time() - t0:.1f}s", flush=True)
    np.savez_compressed(os.path.join(HERE, "referee_batch.npz"), hi=res_hi, lo=res_lo,
                        abs_sum=absum, digests=dig)


def gen_full52():
    c = _cases("range_n52.npz")["n52s3"]
    at, dg, nh = engine._prepare(c["A"], False)
    t0 = time.time()
    hi, lo, sa = R.sum_range(at, dg, nh, 1, 1 << nh, False)
    print(f"full n52s3: {hi} + {lo} cond {sa / abs(hi):.2e} ({time.time() - t0:.0f}s)", flush=True)
    np.savez_compressed(os.path.join(HERE, "referee_full52.npz"), A=c["A"], hi=np.array(hi),
                        lo=np.array(lo), abs_sum=np.array(sa), seconds=np.array(time.time() - t0))


if __name__ == "__main__":
    which = sys.argv[1:] or ["small", "ranges", "batch"]
    if "small" in which or "ranges" in which:
        out = {}
        path = os.path.join(HERE, "referee.npz")
        if os.path.exists(path):
            g = np.load(path)
            out = {k: g[k] for k in g.files}
        if "small" in which:
            gen_small(out)
        if "ranges" in which:
            gen_ranges(out)
        np.savez_compressed(path, **out)
    if "batch" in which:
        gen_batch()
    if "full" in which:
        gen_full52()
