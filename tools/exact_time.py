"""Time the exact GF(p) mode: cfg3 (n=40) and a 0/1 n=52 graph."""
import sys
import time

sys.path.insert(0, ".")

import numpy as np

from paper_1805_12498_b200 import exact, kernels, workloads


def run(name, a, loops=False):
    f = exact.loop_hafnian_exact if loops else exact.hafnian_exact
    f(np.ones((4, 4), int))
    t = time.perf_counter()
    v = f(a)
    dt = time.perf_counter() - t
    n = len(a)
    rows = exact._as_int_matrix(a)
    primes = exact._PRIMES[:1]
    perm = [i ^ 1 for i in range(n)]
    at = np.array([[[rows[perm[i]][j] % p if perm[i] != j else 0 for j in range(n)] for i in range(n)] for p in primes], np.uint32)
    dg = np.zeros((1, n), np.uint32)
    _, ms = kernels.modp_sums(at, dg, primes, n // 2, 1, 1 << (n // 2), loops)
    print(f"{name}: value={v} wall={dt:.3f}s device_ms_per_prime={ms:.1f} terms/s/prime={((1 << (n // 2)) - 1) / ms * 1e3:.3e}", flush=True)


run("cfg3", workloads.cfg3())
rng = np.random.default_rng(5)
adj = np.triu((rng.uniform(size=(52, 52)) < 0.5).astype(np.int64), 1)
run("er52", adj + adj.T)
