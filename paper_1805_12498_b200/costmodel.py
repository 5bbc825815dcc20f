"""Algorithmic cost model of the subset sum and the LPT shard planner.

FLOP model: one complex multiply-add (CMA) = 4 DFMA = 8 FLOP;
only these terms are credited (divisions, pivot search, gathers and redundant
work such as the reference's O(D^3) Horner exp are not):

    CMA(s, D) = sum_{k=1}^{s-2} k(k+1+s)            Hessenberg
              + sum_{k=1}^{s} (k + k(k-1)/2)          charpoly
              + q(q-1)/2 + q,  q = min(D, s)          Newton
              + max(D-s, 0) * s                       Cayley-Hamilton recurrence
              + D(D+1)/2                              exp (recurrence form)
              + [loops] (D-1) s^2 + D s               loop chain

for a subset of size s = 2m.  The same model is the per-range cost used to
shard ranges across GPUs (longest-processing-time-first), which is what the
reference's round-robin dealing gets wrong (SURVEY.md finding 5).
"""

from __future__ import annotations

from functools import lru_cache
from math import comb


def cma(s: int, D: int, loops: bool = False) -> int:
    hess = sum(k * (k + 1 + s) for k in range(1, s - 1))
    cp = sum(k + k * (k - 1) // 2 for k in range(1, s + 1))
    q = min(D, s)
    newton = q * (q - 1) // 2 + q
    rec = max(D - s, 0) * s
    ex = D * (D + 1) // 2
    lp = ((D - 1) * s * s + D * s) if loops else 0
    return hess + cp + newton + rec + ex + lp


def flops_per_popcount(D: int, loops: bool = False) -> list[int]:
    """FLOP of one subset of popcount m, m = 0..D (m = 0 is never evaluated)."""
    return [0] + [8 * cma(2 * m, D, loops) for m in range(1, D + 1)]


@lru_cache(maxsize=None)
def _binom_table(D: int):
    return [[comb(b, p) for p in range(D + 2)] for b in range(D + 2)]


def count_below(x: int, p: int, D: int) -> int:
    """# of integers y in [0, x) with popcount(y) == p (x <= 2^D)."""
    if p < 0:
        return 0
    C = _binom_table(D)
    total, ones = 0, 0
    for b in range(D, -1, -1):
        if (x >> b) & 1:
            need = p - ones
            if 0 <= need <= b:
                total += C[b][need]
            ones += 1
            if ones > p:
                break
    return total


def popcount_histogram(lo: int, hi: int, D: int) -> list[int]:
    """h[p] = # masks in [lo, hi) with popcount p."""
    return [count_below(hi, p, D) - count_below(lo, p, D) for p in range(D + 1)]


def range_bounds(n_half: int, n_ranges: int) -> list[tuple[int, int]]:
    """The reference's fixed ranges [1 + r w, min(1 + (r+1) w, 2^D)) (_numba.py:362-372)."""
    total = 1 << n_half
    w = -(-(total - 1) // n_ranges)
    out = []
    for r in range(n_ranges):
        a = min(1 + r * w, total)
        b = min(a + w, total)
        out.append((a, b))
    return out


def flops_of_range(lo: int, hi: int, D: int, loops: bool = False) -> int:
    h = popcount_histogram(lo, hi, D)
    f = flops_per_popcount(D, loops)
    return sum(h[p] * f[p] for p in range(1, D + 1))


def flops_total(D: int, loops: bool = False) -> int:
    f = flops_per_popcount(D, loops)
    return sum(comb(D, m) * f[m] for m in range(1, D + 1))


def range_costs(n_half: int, n_ranges: int, loops: bool = False) -> list[int]:
    return [flops_of_range(a, b, n_half, loops) for a, b in range_bounds(n_half, n_ranges)]


def lpt_shards(costs, k: int) -> list[list[int]]:
    """Longest-processing-time-first assignment of items to k bins; each bin's
    item list is returned sorted (the device processes ranges in index order).
    Deterministic: ties broken by item index, then bin index."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    loads = [0] * k
    bins: list[list[int]] = [[] for _ in range(k)]
    for i in order:
        b = min(range(k), key=lambda j: (loads[j], j))
        bins[b].append(i)
        loads[b] += costs[i]
    return [sorted(x) for x in bins]


def imbalance(costs, shards) -> float:
    loads = [sum(costs[i] for i in s) for s in shards]
    mean = sum(loads) / len(loads)
    return max(loads) / mean if mean else 1.0
