"""Loop-hafnian timing (dev tool): FAST charpoly on cfg2-like matrices of size n.

    python tools/loop_time.py [n ...]
"""
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

from paper_1805_12498_b200 import engine, workloads as W  # noqa: E402

for n in [int(a) for a in sys.argv[1:]] or [32, 40, 48]:
    A = W.cfg2(n=n)
    for arith in ("fast", "mirror") if n <= 44 else ("fast",):
        engine.loop_hafnian(A, backend="charpoly", arith=arith)
        t = time.perf_counter()
        r = engine.loop_hafnian(A, backend="charpoly", arith=arith)
        dt = time.perf_counter() - t
        h = engine.hafnian(A, backend="charpoly", arith=arith)
        t = time.perf_counter()
        h = engine.hafnian(A, backend="charpoly", arith=arith)
        dh = time.perf_counter() - t
        print(f"n={n} {arith}: loop_hafnian {dt * 1e3:.1f} ms ({(2 ** (n // 2) - 1) / dt:.3e} terms/s), "
              f"hafnian {dh * 1e3:.1f} ms, ratio {dt / dh:.2f}", flush=True)
