import sys; sys.path.insert(0,'.')
import numpy as np
from paper_1805_12498_b200 import engine, exact, kernels
rng = np.random.default_rng(7)
adj = np.triu((rng.uniform(size=(36, 36)) < 0.3).astype(np.int64), 1)
a = adj + adj.T
count = exact.hafnian_exact(a)
for ar in ("fast", "mirror"):
    got = engine.hafnian(a.astype(np.complex128), backend="charpoly", arith=ar)
    print(ar, got, count, abs(got.real-count)/count)
at, dg, nh = engine._prepare(a.astype(np.complex128), False)
masks = np.arange(1, 1 << nh, dtype=np.uint64)
tf, sf = kernels.terms(at, dg, nh, masks, 1, False, arith="fast")
tm, sm = kernels.terms(at, dg, nh, masks, 1, False, arith="mirror")
pc = np.array([bin(int(m)).count('1') for m in masks])
err = np.abs(tf - tm)
print("sum|t|", np.abs(tm).sum(), "statuses", sf.max(), sm.max())
for m in range(1, nh + 1):
    sel = pc == m
    if sel.any():
        print(m, 2*m, "max abs err", err[sel].max(), "max |t|", np.abs(tm[sel]).max(), "sum err", abs((tf[sel]-tm[sel]).sum()))
