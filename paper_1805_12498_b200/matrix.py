"""Input semantics of the hot path: validation, symmetrisation, pair swap.

Host-side mirror of the reference's data layer on the call path
(pkg/src/hafnium/matrix.py:24-157): strict symmetry check with upper->lower
mirroring, the frozen matrix type, pair subsets and the pair swap X.A.
File I/O (matrix.py:177-340) is CLI plumbing and out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import AsymmetricInput, DimensionMismatch, NonSquare, OddDimension

SYMMETRY_RTOL = 1e-12  # matrix.py:24


@dataclass(frozen=True)
class ComplexSymmetricMatrix:
    """n x n complex matrix with exact entry[i,j] == entry[j,i] (matrix.py:30-50)."""

    entries: np.ndarray = field(repr=False)

    def __post_init__(self):
        self.entries.setflags(write=False)

    @property
    def n(self) -> int:
        return self.entries.shape[0]

    def array(self) -> np.ndarray:
        return self.entries.copy()


@dataclass(frozen=True)
class PairSubset:
    """Bitmask over the n/2 pairs; bit i selects pair (2i, 2i+1) (matrix.py:53-83)."""

    mask: int
    width: int

    def __post_init__(self):
        if not 0 <= self.mask < (1 << self.width):
            raise ValueError(f"mask {self.mask:#x} does not fit in {self.width} bits")

    @property
    def cardinality(self) -> int:
        return bin(self.mask).count("1")

    def pair_indices(self) -> list[int]:
        return [i for i in range(self.width) if self.mask >> i & 1]

    def vertex_indices(self) -> np.ndarray:
        idx = np.empty(2 * self.cardinality, dtype=np.int64)
        for j, i in enumerate(self.pair_indices()):
            idx[2 * j] = 2 * i
            idx[2 * j + 1] = 2 * i + 1
        return idx

    @classmethod
    def full(cls, width: int) -> "PairSubset":
        return cls((1 << width) - 1, width)


def _as_array(raw) -> np.ndarray:
    a = np.asarray(raw, dtype=np.complex128)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise NonSquare(f"expected a square matrix, got shape {a.shape}")
    return a


def validate_or_symmetrize(raw, mode: str = "strict") -> ComplexSymmetricMatrix:
    """Strict: accept iff max|A - A^T| <= 1e-12 max(1, max|A|), then mirror the
    upper triangle onto the lower one; auto: average with the transpose
    (matrix.py:93-115)."""
    a = _as_array(raw)
    if mode == "auto":
        a = (a + a.T) / 2
    elif mode == "strict":
        if a.size:
            dev = np.abs(a - a.T).max()
            tol = SYMMETRY_RTOL * max(1.0, float(np.abs(a).max()))
            if dev > tol:
                raise AsymmetricInput(f"max|A - A^T| = {dev:.3e} exceeds tolerance {tol:.3e}")
        a = a.copy()
        iu = np.triu_indices(a.shape[0], k=1)
        a[(iu[1], iu[0])] = a[iu]
    else:
        raise ValueError(f"unknown mode {mode!r}")
    return ComplexSymmetricMatrix(np.ascontiguousarray(a))


def coerce(A, mode: str = "strict") -> ComplexSymmetricMatrix:
    if isinstance(A, ComplexSymmetricMatrix):
        return A
    return validate_or_symmetrize(A, mode=mode)


def pair_swap(A) -> np.ndarray:
    """Rows 2i <-> 2i+1 exchanged: X.A (matrix.py:136-146)."""
    a = A.entries if isinstance(A, ComplexSymmetricMatrix) else np.asarray(A, dtype=np.complex128)
    n = a.shape[0]
    if n % 2:
        raise OddDimension(f"pair swap needs even dimension, got {n}")
    perm = np.arange(n)
    perm[0::2] += 1
    perm[1::2] -= 1
    return np.ascontiguousarray(a[perm])


def pair_submatrix(M, Z: PairSubset) -> np.ndarray:
    a = M.entries if isinstance(M, ComplexSymmetricMatrix) else np.asarray(M, dtype=np.complex128)
    idx = Z.vertex_indices()
    if idx.size and idx[-1] >= a.shape[0]:
        raise DimensionMismatch(f"pair subset selects index {int(idx[-1])} beyond size {a.shape[0]}")
    return np.ascontiguousarray(a[np.ix_(idx, idx)])
