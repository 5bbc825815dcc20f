"""One FAST range pass of the n=52 parity range (ncu target; dev tool)."""
import sys

sys.path.insert(0, '.')
from paper_1805_12498_b200 import engine, kernels, workloads as W  # noqa: E402

A = W.cfg4(3, 52)
at, dg, nh = engine._prepare(A, False)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for _ in range(reps):
    s, f = kernels.sum_mask_range(at, dg, nh, 0, 1 << 20, 512, 1, False, arith="fast")
print(engine.tree_reduce(s))
