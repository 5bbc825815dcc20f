"""Small FAST + MIRROR workload touching every kernel variant (compute-sanitizer target)."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
from paper_1805_12498_b200 import engine, kernels  # noqa: E402

rng = np.random.default_rng(0)
n = 44
g = rng.normal(0, 0.7, (n, n)) + 1j * rng.normal(0, 0.7, (n, n))
a = (g + g.T) / 2 / np.sqrt(n)
at, dg, nh = engine._prepare(a, False)
masks = []
for m in range(1, nh + 1):
    for _ in range(40):
        masks.append(int(sum(1 << int(b) for b in rng.choice(nh, size=m, replace=False))))
masks = np.array(masks, dtype=np.uint64)
for arith in ("fast", "mirror"):
    t, st = kernels.terms(at, dg, nh, masks, 1, False, arith=arith)
    print(arith, "terms", t.size, "status max", int(st.max()))
# loops path and a small full hafnian (staged gathers, class walk)
b = a[:24, :24].copy()
np.fill_diagonal(b, rng.normal(size=24))
print("lhaf", engine.loop_hafnian(b, backend="charpoly", arith="fast"))
print("haf", engine.hafnian(a[:20, :20], backend="charpoly", arith="fast"))
