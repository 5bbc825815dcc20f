import sys, time
sys.path.insert(0, '.')
from paper_1805_12498_b200 import engine, kernels, workloads as W
for name, A, loops, lohi in [("cfg0", W.cfg0(), False, None), ("cfg2", W.cfg2(), True, None), ("cfg3", W.cfg3(), False, None), ("n52range", W.cfg4(3, 52), False, (0, 1 << 20))]:
    at, dg, nh = engine._prepare(A, loops)
    for rep in range(2):
        t = time.perf_counter()
        if lohi:
            s, f = kernels.sum_mask_range(at, dg, nh, lohi[0], lohi[1], 512, 0, loops)
        else:
            s, f = kernels.sum_subsets_det(at, dg, nh, 0, loops, 1, min(512, (1 << nh) - 1))
        dt = time.perf_counter() - t
    print(f"{name} spectral {dt*1e3:.1f} ms result={engine.tree_reduce(s)} fails={int(f.max())}", flush=True)
