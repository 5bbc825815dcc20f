"""cfg1 batch (4096 x n=24) through hafnian_batch: wall time split (dev tool)."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

from paper_1805_12498_b200 import engine, workloads as W  # noqa: E402

mats = np.stack([W.cfg1(s) for s in range(4096)])
arith = sys.argv[1] if len(sys.argv) > 1 else "fast"
for rep in range(3):
    t = time.perf_counter()
    res = engine.hafnian_batch(mats, backend="charpoly", arith=arith)
    dt = time.perf_counter() - t
print(f"batch {arith} {dt*1e3:.1f} ms")
