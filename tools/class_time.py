"""One full n=52 hafnian through one kernel family (for ncu launch lists / metrics).

    python tools/class_time.py [fast|mirror|modp] [n]
"""
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

from paper_1805_12498_b200 import engine, exact, kernels, workloads as W  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "fast"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 52
if mode == "modp":
    rng = np.random.default_rng(5)
    adj = np.triu((rng.uniform(size=(n, n)) < 0.5).astype(np.int64), 1)
    rows = (adj + adj.T).tolist()
    p = exact._PRIMES[:1]
    perm = [i ^ 1 for i in range(n)]
    at = np.array([[[rows[perm[i]][j] % q for j in range(n)] for i in range(n)] for q in p], np.uint32)
    res, ms = kernels.modp_sums(at, np.zeros((1, n), np.uint32), p, n // 2, 1, 1 << (n // 2), False)
    print(res, ms)
else:
    A = W.cfg4(3, n)
    at, dg, nh = engine._prepare(A, False)
    s, f = kernels.sum_subsets_det(at, dg, nh, 1, False, 1, 512, arith=mode)
    print(engine.tree_reduce(s))
