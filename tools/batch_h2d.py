import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1805_12498_b200 import engine, kernels, workloads as W
mats = np.stack([W.cfg1(s) for s in range(4096)])
print("bytes", mats.nbytes)
x = torch.empty(1, device="cuda")
for r in range(3):
    torch.cuda.synchronize(); t = time.perf_counter(); y = torch.from_numpy(mats).to("cuda"); torch.cuda.synchronize(); print("pageable H2D", (time.perf_counter()-t)*1e3, "ms")
pin = torch.from_numpy(mats).pin_memory()
for r in range(3):
    torch.cuda.synchronize(); t = time.perf_counter(); y = pin.to("cuda", non_blocking=True); torch.cuda.synchronize(); print("pinned H2D", (time.perf_counter()-t)*1e3, "ms")
for r in range(3):
    t = time.perf_counter(); res = engine.hafnian_batch(mats, backend="charpoly", arith="fast"); print("batch", (time.perf_counter()-t)*1e3, "ms")
