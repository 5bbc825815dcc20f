"""8-way LPT shard efficiency on one GPU for a library build (HAFB200_LIB=...) (dev tool)."""
import os
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1805_12498_b200 import _lib, costmodel, engine, workloads as W  # noqa: E402

lib = _lib.load(require_device=True)
torch.cuda.set_device(0)
stream = torch.cuda.current_stream()
at, dg, nh = engine._prepare(W.cfg4(3, 52), False)
prob = bench.DeviceProblem(lib, at, dg, nh, False, 0, stream)
costs = costmodel.range_costs(nh, 512)
full = prob.time_ms(list(range(512)), "fast", 2)
ts = [prob.time_ms(s, "fast", 1) for s in costmodel.lpt_shards(costs, 8)]
print(f"{os.environ.get('HAFB200_LIB', 'in-tree')}: full {full:.1f} ms, 8 shards max {max(ts):.1f} sum {sum(ts):.1f} "
      f"eff {full / (8 * max(ts)):.3f}", flush=True)
