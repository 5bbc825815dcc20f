"""A/B timing of a library build (HAFB200_LIB=...): the full n=52 FAST hafnian, best of
3 after a warm-up, plus optional n (dev tool).

    HAFB200_LIB=build_variants/x.so python tools/ab_time.py [n]
"""
import os
import sys
import time

sys.path.insert(0, '.')
from paper_1805_12498_b200 import engine, kernels, workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 52
A = W.cfg4(3, n)
at, dg, nh = engine._prepare(A, False)
kernels.sum_subsets_det(at, dg, nh, 1, False, 1, 512, arith="fast")
ts = []
for _ in range(3):
    t = time.perf_counter()
    s, f = kernels.sum_subsets_det(at, dg, nh, 1, False, 1, 512, arith="fast")
    ts.append(time.perf_counter() - t)
print(f"{os.environ.get('HAFB200_LIB', 'in-tree')}: n={n} best {min(ts) * 1e3:.1f} ms  all {[round(x * 1e3, 1) for x in ts]}  "
      f"result {engine.tree_reduce(s)}", flush=True)
