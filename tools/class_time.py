"""One full n=52 FAST hafnian (for an ncu launch list: per-class kernel times)."""
import sys

sys.path.insert(0, '.')
from paper_1805_12498_b200 import engine, kernels, workloads as W  # noqa: E402

A = W.cfg4(3, 52)
at, dg, nh = engine._prepare(A, False)
s, f = kernels.sum_subsets_det(at, dg, nh, 1, False, 1, 512, arith="fast")
print(engine.tree_reduce(s))
