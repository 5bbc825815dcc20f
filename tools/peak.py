import ctypes, sys
sys.path.insert(0, '.')
from paper_1805_12498_b200 import _lib
L = _lib.load(require_device=True)
for _ in range(3):
    t = ctypes.c_double(); ms = ctypes.c_double()
    _lib.check(L.hafb_fp64_peak(0, ctypes.byref(t), ctypes.byref(ms)))
    print(f"fp64 peak {t.value:.2f} TFLOP/s ({ms.value:.1f} ms)")
