"""Per-rank efficiency of shard shapes on one GPU (dev tool): the full n=52 step, LPT
shards (scattered ranges) and contiguous cost-balanced shards (one mask interval each),
each timed alone; efficiency = full / (k x slowest shard)."""
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1805_12498_b200 import _lib, costmodel, engine  # noqa: E402

lib = _lib.load(require_device=True)
torch.cuda.set_device(0)
stream = torch.cuda.current_stream()
A = bench.workload.__globals__["W"].cfg4(3, 52) if hasattr(bench, "W") else None
from paper_1805_12498_b200 import workloads as W  # noqa: E402
A = W.cfg4(3, 52)
at, dg, nh = engine._prepare(A, False)
prob = bench.DeviceProblem(lib, at, dg, nh, False, 0, stream)
costs = costmodel.range_costs(nh, 512)
full = prob.time_ms(list(range(512)), "fast", 2)
print(f"full {full:.1f} ms")


def contiguous(costs, k):
    pre = np.cumsum(costs)
    tot = pre[-1]
    cuts = [0] + [int(np.searchsorted(pre, tot * i / k)) for i in range(1, k)] + [len(costs)]
    return [list(range(cuts[i], cuts[i + 1])) for i in range(k)]


for k in (2, 4, 8):
    for name, shards in (("lpt", costmodel.lpt_shards(costs, k)), ("contig", contiguous(costs, k))):
        ts = [prob.time_ms(s, "fast", 1) for s in shards]
        imb = costmodel.imbalance(costs, shards)
        print(f"k={k} {name:6s} eff {full / (k * max(ts)):.3f}  sum/full {sum(ts) / full:.3f}  cost imbalance {imb:.4f}  "
              f"shard ms {[round(t, 1) for t in ts]}", flush=True)
