"""FAST vs the reference's own result on the identical ranges [0, 2^20) of the golden
n >= 48 cases: relative and sum|t|-normalised error (dev tool, GPU)."""
import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np  # noqa: E402
from conftest import load_golden, rel_err  # noqa: E402
from paper_1805_12498_b200 import engine, kernels  # noqa: E402
r = load_golden("range_n52.npz")
for name, case in r.items():
    at, dg, nh = engine._prepare(case["A"], False)
    sums, fails = kernels.sum_mask_range(at, dg, nh, 0, 1 << 20, 512, 1, False, arith="fast")
    t, _ = kernels.terms(at, dg, nh, np.arange(1, 1 << 20, dtype=np.uint64), 1, False, arith="fast")
    ref = complex(case["result_b1"])
    got = engine.tree_reduce(sums)
    print(f"{name}: rel {rel_err(got, ref):.3e}  sum|t|-normalised {abs(got - ref) / np.abs(t).sum():.3e}  "
          f"cond {np.abs(t).sum() / abs(ref):.2e}")
