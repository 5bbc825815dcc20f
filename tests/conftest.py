import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def random_symmetric(n, seed, diag_scale=1.0):
    """Seeded complex symmetric matrix, entries in the unit square (reference tests/conftest.py:5-12)."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
    a = (a + a.T) / 2
    if diag_scale != 1.0:
        np.fill_diagonal(a, diag_scale * np.diag(a))
    return a


def rel_err(approx, exact):
    exact = complex(exact)
    scale = max(1e-300, abs(exact))
    return abs(complex(approx) - exact) / scale


def bits(a):
    """Raw bit pattern of complex128 data, for bit-identity assertions."""
    return np.ascontiguousarray(a, dtype=np.complex128).view(np.uint64)


def digest(A) -> int:
    """8-byte fingerprint of a matrix's exact bits.  cfg1 inputs go through LAPACK QR,
    which may differ in the last ulp on another CPU: tests regenerate the batch and
    compare digests with the fixture's before demanding bit-identity."""
    import hashlib

    h = hashlib.blake2b(np.ascontiguousarray(A, np.complex128).tobytes(), digest_size=8)
    return int.from_bytes(h.digest(), "little")


def load_golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} missing")
    z = np.load(path, allow_pickle=False)
    groups = {}
    for key in z.files:
        g, field = key.split("/", 1)
        groups.setdefault(g, {})[field] = z[key]
    return groups


@pytest.fixture
def rng():
    return np.random.default_rng(12345)
