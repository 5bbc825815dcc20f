"""The C-ABI library: loads without a GPU and exports every symbol include/hafb200.h
declares, with the signatures the ctypes binding uses.  No compute calls here."""

import os
import re

from conftest import REPO
from paper_1805_12498_b200 import _lib


def header_symbols():
    text = open(os.path.join(REPO, "include", "hafb200.h")).read()
    return set(re.findall(r"\b(hafb_[a-z0-9_]+)\s*\(", text))


def test_library_loads_and_reports_abi():
    lib = _lib.load(require_device=False)
    assert lib.hafb_abi_version() == _lib.ABI_VERSION


def test_every_header_symbol_exported_and_bound():
    lib = _lib.load(require_device=False)
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert syms == set(_lib.SIGNATURES), syms ^ set(_lib.SIGNATURES)


def test_sass_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_argument_errors_without_device():
    import numpy as np

    lib = _lib.load(require_device=False)
    a = np.zeros((4, 4), np.complex128)
    d = np.zeros(4, np.complex128)
    sums = np.zeros(2, np.complex128)
    fails = np.zeros(2, np.int64)
    rc = lib.hafb_sum_subsets_det(_lib.dptr(a), _lib.dptr(d), 40, 1, 0, 2, 30, 0, 0,
                                  _lib.dptr(sums), _lib.i64ptr(fails))
    assert rc == -1 and b"n_half" in lib.hafb_last_error()
