"""Independent brute-force oracles for small cases.  TEST INFRASTRUCTURE ONLY.

Restates the definitions the reference's own tests use as independent
checks (pkg/src/hafnium/oracle.py:24-188): the hafnian as a sum over perfect
matchings, the loop hafnian over single-pair matchings (pairs and loops), the
permanent by Ryser's formula, the number of matchings of a graph, and the
closed forms (2k-1)!! and the telephone numbers.  Plain recursive Python,
fine for n <= 12.
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np


def double_factorial(k: int) -> int:
    """k!!, with (-1)!! = 0!! = 1 (oracle.py:24-32)."""
    out = 1
    while k > 1:
        out *= k
        k -= 2
    return out


def telephone(n: int) -> int:
    """Involutions of n elements: T(n) = T(n-1) + (n-1) T(n-2) (oracle.py:35-44)."""
    a, b = 1, 1
    for m in range(2, n + 1):
        a, b = b, b + (m - 1) * a
    return b if n >= 1 else 1


def _matchings(vertices: tuple, loops: bool):
    if not vertices:
        yield ()
        return
    v, rest = vertices[0], vertices[1:]
    if loops:
        for m in _matchings(rest, loops):
            yield ((v, v),) + m
    for k, w in enumerate(rest):
        for m in _matchings(rest[:k] + rest[k + 1:], loops):
            yield ((v, w),) + m


def hafnian_bruteforce(A) -> complex:
    """Sum over perfect matchings of the product of matched entries (oracle.py:79-89)."""
    a = np.asarray(A, dtype=np.complex128)
    total = 0.0 + 0.0j
    for m in _matchings(tuple(range(a.shape[0])), False):
        p = 1.0 + 0.0j
        for i, j in m:
            p *= a[i, j]
        total += p
    return complex(total)


def loop_hafnian_bruteforce(A) -> complex:
    """Sum over single-pair matchings, loops weighted by the diagonal (oracle.py:92-102)."""
    a = np.asarray(A, dtype=np.complex128)
    total = 0.0 + 0.0j
    for m in _matchings(tuple(range(a.shape[0])), True):
        p = 1.0 + 0.0j
        for i, j in m:
            p *= a[i, j]
        total += p
    return complex(total)


def permanent_ryser(W) -> complex:
    """Ryser's inclusion-exclusion formula (oracle.py:122-148), plain subset loop."""
    w = np.asarray(W, dtype=np.complex128)
    m = w.shape[0]
    if m == 0:
        return 1.0 + 0.0j
    total = 0.0 + 0.0j
    for s in range(1, 1 << m):
        cols = [j for j in range(m) if s >> j & 1]
        rows = w[:, cols].sum(axis=1)
        total += (-1) ** (m - len(cols)) * np.prod(rows)
    return complex(total)


def matching_count(adjacency) -> int:
    """Number of matchings, including the empty one, of a loopless graph (oracle.py:151-178)."""
    a = np.asarray(adjacency)
    n = a.shape[0]
    adj = [sum(1 << j for j in range(n) if j != i and a[i, j] != 0) for i in range(n)]

    @lru_cache(maxsize=None)
    def count(mask: int) -> int:
        if mask == 0:
            return 1
        v = (mask & -mask).bit_length() - 1
        rest = mask & ~(1 << v)
        total = count(rest)
        nbrs = adj[v] & rest
        while nbrs:
            wb = nbrs & -nbrs
            total += count(rest & ~wb)
            nbrs ^= wb
        return total

    return count((1 << n) - 1)


def bipartite_embedding(W) -> np.ndarray:
    w = np.asarray(W, dtype=np.complex128)
    m = w.shape[0]
    out = np.zeros((2 * m, 2 * m), dtype=np.complex128)
    out[:m, m:] = w
    out[m:, :m] = w.T
    return out


def hafnian_exact_dp(A, loops: bool = False) -> int:
    """Exact (loop) hafnian of an integer matrix with Python ints: the lowest
    remaining vertex is matched to each other remaining vertex (or, with loops,
    to itself), memoised over the remaining-vertex bitmask.  O(2^n n); n <= 20.
    Independent of the subset-sum formula (checks the exact GF(p) mode)."""
    rows = [[int(v) for v in r] for r in np.asarray(A, dtype=object).tolist()] if len(A) else []
    n = len(rows)

    @lru_cache(maxsize=None)
    def rec(rem: int) -> int:
        if rem == 0:
            return 1
        i = (rem & -rem).bit_length() - 1
        rest = rem & ~(1 << i)
        total = rows[i][i] * rec(rest) if loops else 0
        r = rest
        while r:
            j = (r & -r).bit_length() - 1
            r &= r - 1
            if rows[i][j]:
                total += rows[i][j] * rec(rest & ~(1 << j))
        return total

    if n % 2 and not loops:
        return 0
    return rec((1 << n) - 1)
