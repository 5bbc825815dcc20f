import sys
sys.path.insert(0, '.')
import torch
import bench
from paper_1805_12498_b200 import _lib, costmodel, engine, workloads as W
lib = _lib.load(require_device=True)
torch.cuda.set_device(0)
stream = torch.cuda.current_stream()
A = W.cfg4(3, 52)
at, dg, nh = engine._prepare(A, False)
prob = bench.DeviceProblem(lib, at, dg, nh, False, 0, stream)
costs = costmodel.range_costs(nh, 512)
sh = costmodel.lpt_shards(costs, 8)[0]
prob.launch(list(range(512)), "fast"); torch.cuda.synchronize()
prob.launch(sh, "fast"); torch.cuda.synchronize()
