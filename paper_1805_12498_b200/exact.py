"""Exact hafnian / loop hafnian of INTEGER matrices.

The reference returns a complex128 for every input, so integer hafnians beyond
2^53 come back rounded (cfg3, the 0/1 adjacency matrix of a 40-vertex graph:
the reference returns 3.0854435799026726e17 for the count 308544357990268074,
SURVEY.md finding 4).  Here the same subset-sum formula (engine.py:153-178,
per-subset steps _numba.py:36-351) runs in GF(p) on the device for a few primes
p < 2^31 (kernel csrc/term_modp.cuh behind ``hafb_modp_sums``) and the residues
are lifted to the exact integer by the Chinese remainder theorem.  Enough primes
are used that their product exceeds twice an a-priori bound on |haf(A)|, so the
centred lift is the hafnian itself, not a guess.

Input semantics follow the float API where they apply: a square, even-sized,
exactly symmetric integer matrix (``AsymmetricInput`` otherwise); the hafnian
ignores the diagonal; n = 0 gives 1.  Entries may be arbitrary Python ints.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from numbers import Integral

import numpy as np

from . import costmodel, kernels
from .errors import AsymmetricInput, NonSquare, OddDimension, TooLarge

PRIME_LIMIT = 1 << 31


def _is_prime(x: int) -> bool:
    """Deterministic Miller-Rabin for x < 3.4e14 (bases 2, 3, 5, 7, 11, 13, 17)."""
    if x < 2:
        return False
    for q in (2, 3, 5, 7, 11, 13, 17):
        if x % q == 0:
            return x == q
    d, s = x - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in (2, 3, 5, 7, 11, 13, 17):
        y = pow(a, d, x)
        if y in (1, x - 1):
            continue
        for _ in range(s - 1):
            y = y * y % x
            if y == x - 1:
                break
        else:
            return False
    return True


def primes_below(limit: int, count: int) -> list[int]:
    """The `count` largest primes below `limit`, descending."""
    out, x = [], limit - 1
    while len(out) < count:
        if _is_prime(x):
            out.append(x)
        x -= 1
    return out


_PRIMES = primes_below(PRIME_LIMIT, 64)


def _double_factorial(k: int) -> int:
    out = 1
    while k > 1:
        out *= k
        k -= 2
    return out


def _telephone(n: int) -> int:
    a, b = 1, 1
    for m in range(2, n + 1):
        a, b = b, b + (m - 1) * a
    return b


def hafnian_bound(A: list[list[int]], loops: bool) -> int:
    """|haf(A)| <= #matchings * (max entry)^(factors): (n-1)!! amax^(n/2) for the
    hafnian, T(n) max(1, amax, dmax)^n for the loop hafnian."""
    n = len(A)
    if n == 0:
        return 1
    amax = max((abs(A[i][j]) for i in range(n) for j in range(n) if i != j), default=0)
    if not loops:
        return _double_factorial(n - 1) * amax ** (n // 2)
    dmax = max(abs(A[i][i]) for i in range(n))
    return _telephone(n) * max(1, amax, dmax) ** n


def _as_int_matrix(A) -> list[list[int]]:
    """Exact integer entries as Python ints (ints, integer numpy dtypes, or float /
    complex entries that are exactly integral and real)."""
    if isinstance(A, np.ndarray) and A.dtype.kind in "iu":
        rows = A.tolist()
    else:
        arr = np.asarray(A, dtype=object)
        if arr.ndim != 2:
            raise NonSquare(f"expected a square matrix, got shape {arr.shape}")
        rows = []
        for row in arr.tolist():
            out = []
            for v in row:
                if isinstance(v, (bool, np.bool_)):
                    v = int(v)
                if isinstance(v, Integral):
                    out.append(int(v))
                    continue
                c = complex(v)
                if c.imag != 0.0 or not float(c.real).is_integer():
                    raise ValueError(f"exact mode needs integer entries, got {v!r}")
                out.append(int(c.real))
            rows.append(out)
    n = len(rows)
    if any(len(r) != n for r in rows):
        raise NonSquare(f"expected a square matrix, got {n} rows of lengths {sorted({len(r) for r in rows})}")
    for i in range(n):
        for j in range(i + 1, n):
            if rows[i][j] != rows[j][i]:
                raise AsymmetricInput(f"exact mode needs an exactly symmetric matrix: A[{i},{j}] != A[{j},{i}]")
    return rows


def _crt(residues: list[int], primes: list[int]) -> int:
    """Centred CRT lift: the unique x with |x| < prod(p)/2 and x = r_i mod p_i."""
    M = 1
    for p in primes:
        M *= p
    x = 0
    for r, p in zip(residues, primes):
        Mi = M // p
        x += int(r) * Mi * pow(Mi, -1, p)
    x %= M
    return x - M if x > M // 2 else x


def _contiguous_shards(n_half: int, devices: int) -> list[tuple[int, int]]:
    """[lo, hi) mask intervals of about equal cost (the exact sum is order-free)."""
    bounds = costmodel.range_bounds(n_half, 512)
    costs = costmodel.range_costs(n_half, 512)
    total = sum(costs)
    out, start, acc = [], bounds[0][0], 0
    k = 0
    for i, c in enumerate(costs):
        acc += c
        if k < devices - 1 and acc >= total * (k + 1) / devices:
            out.append((start, bounds[i][1]))
            start = bounds[i][1]
            k += 1
    out.append((start, 1 << n_half))
    return [s for s in out if s[1] > s[0]]


def _exact(A, loops: bool, devices: int | None, n_primes: int | None) -> int:
    rows = _as_int_matrix(A)
    n = len(rows)
    if n == 0:
        return 1
    if n % 2:
        raise OddDimension(f"hafnian needs even dimension, got n={n}")
    n_half = n // 2
    if n_half > kernels.MAX_HALF:
        raise TooLarge(f"n={n} exceeds the device engine's limit n <= {2 * kernels.MAX_HALF}")
    if not loops:
        for i in range(n):
            rows[i][i] = 0
    bound = hafnian_bound(rows, loops)
    if n_primes is None:
        n_primes, prod = 0, 1
        while prod <= 2 * bound:
            prod *= _PRIMES[n_primes]
            n_primes += 1
    primes = _PRIMES[:n_primes]
    perm = [i ^ 1 for i in range(n)]  # X.A: rows 2i <-> 2i+1 (matrix.py:136-146)
    at = np.empty((n_primes, n, n), np.uint32)
    dg = np.empty((n_primes, n), np.uint32)
    for k, p in enumerate(primes):
        at[k] = [[rows[perm[i]][j] % p for j in range(n)] for i in range(n)]
        dg[k] = [rows[i][i] % p for i in range(n)]
    devices = max(1, int(devices or 1))
    shards = _contiguous_shards(n_half, devices) if devices > 1 else [(1, 1 << n_half)]

    def run(d):
        lo, hi = shards[d]
        res, _ = kernels.modp_sums(at, dg, primes, n_half, lo, hi, loops, device=d)
        return res

    if len(shards) == 1:
        parts = [run(0)]
    else:
        with ThreadPoolExecutor(max_workers=len(shards)) as ex:
            parts = list(ex.map(run, range(len(shards))))
    residues = [sum(int(r[k]) for r in parts) % p for k, p in enumerate(primes)]
    return _crt(residues, primes)


def hafnian_exact(A, *, devices: int | None = None, n_primes: int | None = None) -> int:
    """Exact hafnian of an integer symmetric matrix (Python int)."""
    return _exact(A, False, devices, n_primes)


def loop_hafnian_exact(A, *, devices: int | None = None, n_primes: int | None = None) -> int:
    """Exact loop hafnian of an integer symmetric matrix (Python int)."""
    return _exact(A, True, devices, n_primes)
