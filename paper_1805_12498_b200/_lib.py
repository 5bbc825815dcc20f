"""ctypes binding of libhafb200.so (include/hafb200.h).

The library is built in-tree (paper_1805_12498_b200/build.py).  There is no
CPU fallback: if the library is missing or no CUDA device is visible, every
compute call raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import DeviceError

_HERE = os.path.dirname(os.path.abspath(__file__))
# HAFB200_LIB overrides the in-tree library (dev: A/B timing of build variants)
LIB_PATH = os.environ.get("HAFB200_LIB") or os.path.join(_HERE, "libhafb200.so")
ABI_VERSION = 1

_lock = threading.Lock()
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_vp = ctypes.c_void_p
_int, _u64, _i64, _size = ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_size_t

# name -> (restype, argtypes); every symbol include/hafb200.h declares
SIGNATURES = {
    "hafb_abi_version": (_int, []),
    "hafb_last_error": (ctypes.c_char_p, []),
    "hafb_device_count": (_int, []),
    "hafb_sum_subsets_det": (_int, [_dp, _dp, _int, _int, _int, _int, _int, _int, _int, _dp, _i64p]),
    "hafb_sum_subsets_fast": (_int, [_dp, _dp, _int, _int, _int, _int, _int, _int, _int, _int, _dp,
                                     _i64p]),
    "hafb_sum_mask_range": (_int, [_dp, _dp, _int, _u64, _u64, _int, _int, _int, _int, _int, _int,
                                   _dp, _i64p]),
    "hafb_terms": (_int, [_dp, _dp, _int, _u64p, _i64, _int, _int, _int, _int, _int, _dp, _i32p]),
    "hafb_batch": (_int, [_dp, _dp, _int, _int, _int, _int, _int, _int, _int, _int, _dp, _i64p]),
    "hafb_power_traces": (_int, [_dp, _int, _int, _int, _int, _int, _int, _dp, _i64p, _i32p]),
    "hafb_charpoly_coefficients": (_int, [_dp, _int, _int, _int, _dp]),
    "hafb_range_workspace_bytes": (_size, [_int, _u64, _u64, _int]),
    "hafb_sum_mask_range_async": (_int, [_vp, _vp, _int, _u64, _u64, _int, _int, _int, _int, _int,
                                         _vp, _size, _vp, _vp, _vp]),
    "hafb_sum_range_list": (_int, [_dp, _dp, _int, _int, _i32p, _int, _int, _int, _int, _int, _int,
                                   _dp, _i64p]),
    "hafb_range_list_workspace_bytes": (_size, [_int, _int, _int]),
    "hafb_sum_range_list_async": (_int, [_vp, _vp, _int, _int, _i32p, _int, _int, _int, _int,
                                         _int, _vp, _size, _vp, _vp, _vp, _vp]),
    "hafb_launch_count": (_i64, [_int]),
    "hafb_trim_pool": (_int, [_int]),
    "hafb_fp64_peak": (_int, [_int, _dp, _dp]),
    "hafb_batch_raw": (_int, [_dp, _int, _int, _int, _int, _int, _int, _int, _int, ctypes.c_double,
                              _dp, _i64p, _i64p, _dp, _dp]),
    "hafb_modp_sums": (_int, [_u32p, _u32p, _u32p, _int, _int, _u64, _u64, _int, _int, _u64p, _dp]),
}


def load(require_device: bool = False):
    """Load (once) and return the library; raise DeviceError if unusable."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DeviceError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_1805_12498_b200.build`"
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.hafb_abi_version() != ABI_VERSION:
                raise DeviceError("libhafb200.so ABI version mismatch; rebuild it")
            _lib = lib
    if require_device and _lib.hafb_device_count() < 1:
        raise DeviceError("no CUDA device visible: the B200 engine has no CPU fallback")
    return _lib


def check(rc: int):
    if rc != 0:
        msg = _lib.hafb_last_error().decode(errors="replace") if _lib is not None else ""
        raise DeviceError(f"libhafb200 call failed (rc={rc}): {msg}")


def c128(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def i64ptr(a: np.ndarray):
    return a.ctypes.data_as(_i64p)


def i32ptr(a: np.ndarray):
    return a.ctypes.data_as(_i32p)


def u64ptr(a: np.ndarray):
    return a.ctypes.data_as(_u64p)
