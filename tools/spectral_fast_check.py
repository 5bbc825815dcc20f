"""FAST spectral backend vs the bit-exact (MIRROR) spectral kernel and the charpoly FAST
path: results and timings on the BASELINE configs (dev tool).

    python tools/spectral_fast_check.py
"""
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

from paper_1805_12498_b200 import engine, kernels, workloads as W  # noqa: E402


def run(at, dg, nh, loops, lohi, arith, backend):
    t = time.perf_counter()
    if lohi is None:
        s, f = kernels.sum_subsets_det(at, dg, nh, backend, loops, 1, min(512, (1 << nh) - 1), arith=arith)
    else:
        s, f = kernels.sum_mask_range(at, dg, nh, lohi[0], lohi[1], 512, backend, loops, arith=arith)
    return engine.tree_reduce(s), int(f.max()), time.perf_counter() - t


rng = np.random.default_rng(7)
cases = [("cfg0", W.cfg0(), False, None), ("cfg2", W.cfg2(), True, None), ("cfg3", W.cfg3(), False, None)]
for n in (6, 10, 16, 24):
    A = (rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))) / np.sqrt(n)
    A = (A + A.T) / 2
    cases.append((f"rand{n}", A, False, None))
    cases.append((f"rand{n}L", A, True, None))
cases += [("n52r16", W.cfg4(3, 52), False, (0, 1 << 16)), ("n52r20", W.cfg4(3, 52), False, (0, 1 << 20))]
for name, A, loops, lohi in cases:
    at, dg, nh = engine._prepare(A, loops)
    out = {}
    for arith, backend in (("mirror", 0), ("fast", 0), ("fast", 1)):
        run(at, dg, nh, loops, lohi, arith, backend)
        out[(arith, backend)] = run(at, dg, nh, loops, lohi, arith, backend)
    ref = out[("mirror", 0)][0]
    fs, fc = out[("fast", 0)][0], out[("fast", 1)][0]
    print(f"{name:8s} mirror-spec {out[('mirror', 0)][2] * 1e3:9.2f} ms  fast-spec {out[('fast', 0)][2] * 1e3:8.2f} ms "
          f"(fails {out[('fast', 0)][1]})  fast-cp {out[('fast', 1)][2] * 1e3:8.2f} ms  "
          f"rel(fast-spec, mirror-spec) {abs(fs - ref) / abs(ref):.2e}  rel(fast-cp, mirror-spec) {abs(fc - ref) / abs(ref):.2e}",
          flush=True)
