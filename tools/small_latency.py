"""Where a small hafnian's wall time goes (dev tool): host preparation, the C call, the tree."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

from paper_1805_12498_b200 import _lib, engine, kernels, workloads as W  # noqa: E402

for n in (8, 12, 20, 24):
    A = W.cfg0() if n == 20 else W.cfg4(3, n)
    for arith in ("fast", "mirror"):
        engine.hafnian(A, backend="charpoly", arith=arith)
        N = 300
        t0 = time.perf_counter()
        for _ in range(N):
            engine.hafnian(A, backend="charpoly", arith=arith)
        t_all = (time.perf_counter() - t0) / N
        t0 = time.perf_counter()
        for _ in range(N):
            at, dg, nh = engine._prepare(A, False)
        t_prep = (time.perf_counter() - t0) / N
        t0 = time.perf_counter()
        for _ in range(N):
            s, f = kernels.sum_subsets_det(at, dg, nh, 1, False, 1, 512, arith=arith)
        t_k = (time.perf_counter() - t0) / N
        lib = _lib.load(require_device=True)
        atc, dgc = _lib.c128(at), _lib.c128(dg)
        sums = np.zeros(512, np.complex128)
        fails = np.zeros(512, np.int64)
        args = (_lib.dptr(atc), _lib.dptr(dgc), int(nh), 1, 0, 512, 30, kernels._arith_id(arith), 0,
                _lib.dptr(sums), _lib.i64ptr(fails))
        try:
            t0 = time.perf_counter()
            for _ in range(N):
                lib.hafb_sum_subsets_det(*args)
            t_c = (time.perf_counter() - t0) / N
        except Exception as e:  # signature drift: report the Python-level numbers only
            t_c = float("nan")
        t0 = time.perf_counter()
        for _ in range(N):
            engine.tree_reduce(s)
        t_tree = (time.perf_counter() - t0) / N
        print(f"n={n} {arith}: hafnian {t_all * 1e6:.0f} us = prepare {t_prep * 1e6:.0f} + kernels.sum_subsets_det "
              f"{t_k * 1e6:.0f} (C call {t_c * 1e6:.0f}) + tree {t_tree * 1e6:.0f}", flush=True)
