"""Where the time of a small problem goes (dev tool): wall time of hafnian() on cfg0 /
cfg2 and of the device range-list call, for an ncu launch list of the same run.

    python tools/small_problem.py [reps]
"""
import sys
import time

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))

from paper_1805_12498_b200 import engine, workloads  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for name, A, loops in (("cfg0", workloads.cfg0(), False), ("cfg2", workloads.cfg2(), True)):
    f = engine.loop_hafnian if loops else engine.hafnian
    f(A, backend="charpoly", arith="fast")
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f(A, backend="charpoly", arith="fast")
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"{name}: median {1e3 * ts[len(ts) // 2]:.3f} ms, min {1e3 * ts[0]:.3f} ms")
