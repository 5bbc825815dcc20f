"""Canonical synthetic inputs for the five BASELINE.json configs.

Seeded numpy ``default_rng`` (PCG64) generators with a fixed draw order, as
fixed by SURVEY.md Appendix A.  BASELINE names no public dataset; these
seeded matrices stand in for it.  Used by bench.py and the tests; the
hot path itself never calls them.
"""

from __future__ import annotations

import math

import numpy as np


def gaussian_symmetric(n: int, seed: int) -> np.ndarray:
    """cfg0 / cfg4 base: A = (G + G^T)/2 with G ~ N(0,1/2) + i N(0,1/2).

    The real block is drawn before the imaginary block.
    """
    rng = np.random.default_rng(seed)
    sd = math.sqrt(0.5)
    g = rng.normal(0.0, sd, (n, n)) + 1j * rng.normal(0.0, sd, (n, n))
    return (g + g.T) / 2


def cfg0(seed: int = 0, n: int = 20) -> np.ndarray:
    return gaussian_symmetric(n, seed)


def cfg1(seed: int, n: int = 24, modes: int = 48) -> np.ndarray:
    """GBS-like: principal submatrix (repeats allowed) of U diag(tanh r) U^T
    with U Haar (QR of a complex Gaussian with the phase fix)."""
    rng = np.random.default_rng(seed)
    z = (rng.normal(size=(modes, modes)) + 1j * rng.normal(size=(modes, modes))) / math.sqrt(2.0)
    q, r = np.linalg.qr(z)
    d = np.diag(r)
    u = q * (d / np.abs(d))[None, :]
    rr = rng.uniform(0.3, 1.0, modes)
    b = (u * np.tanh(rr)[None, :]) @ u.T
    idx = np.sort(rng.integers(0, modes, n))
    return np.ascontiguousarray(b[np.ix_(idx, idx)])


def cfg2(seed: int = 1, n: int = 32) -> np.ndarray:
    """Loop hafnian input: cfg0-style A with diag(A) := d, d ~ N(0,1/2) + i N(0,1/2)
    drawn from the same stream after G."""
    rng = np.random.default_rng(seed)
    sd = math.sqrt(0.5)
    g = rng.normal(0.0, sd, (n, n)) + 1j * rng.normal(0.0, sd, (n, n))
    d = rng.normal(0.0, sd, n) + 1j * rng.normal(0.0, sd, n)
    a = (g + g.T) / 2
    np.fill_diagonal(a, d)
    return a


def cfg3(seed: int = 2, n: int = 40) -> np.ndarray:
    """Erdos-Renyi p=0.5 adjacency, zero diagonal, cast to complex128."""
    rng = np.random.default_rng(seed)
    adj = np.triu((rng.uniform(size=(n, n)) < 0.5).astype(np.int64), k=1)
    return (adj + adj.T).astype(np.complex128)


def cfg4(seed: int = 3, n: int = 52) -> np.ndarray:
    return gaussian_symmetric(n, seed) / math.sqrt(n)


CONFIGS = {
    "cfg0": dict(n=20, loops=False, desc="single hafnian n=20, seed 0"),
    "cfg1": dict(n=24, loops=False, desc="batch of 4096 GBS-like hafnians n=24, seeds 0..4095"),
    "cfg2": dict(n=32, loops=True, desc="loop hafnian n=32, seed 1"),
    "cfg3": dict(n=40, loops=False, desc="ER(0.5) perfect-matching count n=40, seed 2"),
    "cfg4": dict(n=52, loops=False, desc="complex hafnian n=52 (and 56), seeds 3/4, /sqrt(n)"),
}
