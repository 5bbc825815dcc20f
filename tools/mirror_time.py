"""Time one full n=52 MIRROR hafnian (dev tool; HAFB200_LIB selects a library build)."""
import sys
import time

sys.path.insert(0, ".")
from paper_1805_12498_b200 import engine, kernels, workloads as W  # noqa: E402

A = W.cfg4(3, 52)
at, dg, nh = engine._prepare(A, False)
for r in range(2):
    t = time.perf_counter()
    s, f = kernels.sum_subsets_det(at, dg, nh, 1, False, 1, 512, arith="mirror")
    dt = time.perf_counter() - t
print(f"mirror n52 full {dt:.3f} s {engine.tree_reduce(s)!r}")
