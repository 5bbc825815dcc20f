import sys, itertools, numpy as np
sys.path.insert(0, '.')
from paper_1805_12498_b200 import engine, kernels, workloads as W
from oracle import oracle as O
A = W.cfg4(3, 52)
at, dg, nh = engine._prepare(A, False)
D = nh
for m in (17, 18, 19):
    # all masks of popcount m below 2^D, in chunks
    from math import comb
    bad = []
    ms = np.array([sum(1 << b for b in c) for c in itertools.combinations(range(D), m)], dtype=np.uint64)
    t, st = kernels.terms(at, dg, nh, ms, 1, False, arith="fast")
    nb = np.nonzero(st)[0]
    big = np.nonzero(~np.isfinite(t) | (np.abs(t) > 1e3))[0]
    print("m", m, "count", len(ms), "bad status", len(nb), "huge", len(big), flush=True)
    sel = list(nb[:5]) + list(big[:5])
    for i in sel:
        mk = int(ms[i])
        ref, rst = O.subset_term(at, dg, mk, nh, 1, False) if hasattr(O, 'subset_term') else (None, None)
        print(hex(mk), t[i], st[i], "oracle", ref, rst, flush=True)
    # sample compare
    rng = np.random.default_rng(0)
    idx = rng.choice(len(ms), 2000, replace=False)
    refs, _ = O.terms(at, dg, nh, ms[idx], 1, False)
    err = np.abs(t[idx] - refs) / np.maximum(np.abs(refs), 1e-300)
    print("sample max rel err", err.max(), "median", np.median(err), flush=True)
