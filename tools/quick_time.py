"""Ad-hoc device timing of the range driver for the BASELINE configs (dev tool)."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

from paper_1805_12498_b200 import costmodel, engine, kernels, workloads as W  # noqa: E402

cases = [("cfg0", W.cfg0(), False, None), ("cfg2", W.cfg2(), True, None),
         ("cfg3", W.cfg3(), False, None), ("n52range", W.cfg4(3, 52), False, (0, 1 << 20))]
if len(sys.argv) > 1 and sys.argv[1] == "full":
    cases.append(("n52full", W.cfg4(3, 52), False, "full"))
arith_modes = ["fast", "mirror"]
for name, A, loops, lohi in cases:
    at, dg, nh = engine._prepare(A, loops)
    res = {}
    for arith in arith_modes:
        if arith == "mirror" and lohi == "full":
            continue
        for rep in range(2):
            t = time.perf_counter()
            if lohi is None or lohi == "full":
                s, f = kernels.sum_subsets_det(at, dg, nh, 1, loops, 1, min(512, (1 << nh) - 1), arith=arith)
                nt = (1 << nh) - 1
                fl = costmodel.flops_total(nh, loops)
            else:
                s, f = kernels.sum_mask_range(at, dg, nh, lohi[0], lohi[1], 512, 1, loops, arith=arith)
                nt = lohi[1] - lohi[0]
                fl = costmodel.flops_of_range(lohi[0], lohi[1], nh, loops)
            dt = time.perf_counter() - t
        r = engine.tree_reduce(s)
        res[arith] = r
        print(f"{name} {arith:6s} {dt*1e3:9.2f} ms  {nt/dt:.3e} terms/s  {fl/dt/1e12:.3f} TF/s  "
              f"fails={int(f.max())} result={r}", flush=True)
    if "mirror" in res:
        print(f"   rel diff fast vs mirror: {abs(res['fast']-res['mirror'])/abs(res['mirror']):.3e}")

if len(sys.argv) > 1 and sys.argv[-1] in ("batch", "full"):
    # cfg1: batch of 4096 GBS-like hafnians, n = 24
    mats = [W.cfg1(s) for s in range(4096)]
    for arith in ("fast", "mirror"):
        for rep in range(2):
            t = time.perf_counter()
            res = engine.hafnian_batch(mats, backend="charpoly", arith=arith)
            dt = time.perf_counter() - t
        nt = 4096 * 4095
        fl = 4096 * costmodel.flops_total(12)
        print(f"cfg1 batch {arith:6s} {dt*1e3:9.2f} ms  {nt/dt:.3e} terms/s  {fl/dt/1e12:.3f} TF/s  "
              f"res[0]={res[0]}", flush=True)
