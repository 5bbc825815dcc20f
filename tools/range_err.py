import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from conftest import load_golden, rel_err
from paper_1805_12498_b200 import engine, kernels
r = load_golden("range_n52.npz")
for name, case in r.items():
    at, dg, nh = engine._prepare(case["A"], False)
    sums, fails = kernels.sum_mask_range(at, dg, nh, 0, 1 << 20, 512, 1, False, arith="fast")
    print(name, list(case.keys())[:8], rel_err(engine.tree_reduce(sums), complex(case["result_b1"])))
