"""The N>1 path on CPU: world_size 2 and 3 gloo process groups run the same
shard / all-gather / fixed-tree orchestration as the GPU ranks (distributed.py),
with the C oracle computing each rank's range partials.  The result must be
bit-identical to the single-process reference pipeline."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import REPO  # noqa: F401  (sys.path)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, loops, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_1805_12498_b200 import costmodel, distributed, workloads
    from paper_1805_12498_b200.engine import _prepare

    A = workloads.cfg2(n=n) if loops else workloads.cfg0(n=n)
    at, dg, nh = _prepare(A, loops)
    nr, _ = distributed.shard_plan(nh, world, loops=loops)
    bounds = costmodel.range_bounds(nh, nr)

    def partials_fn(ranges):
        s = np.zeros(len(ranges), np.complex128)
        f = np.zeros(len(ranges), np.int64)
        for i, r in enumerate(ranges):
            lo, hi = bounds[r]
            ps, pf = O.sum_mask_range(at, dg, nh, lo, hi, 1, backend=1, include_loops=loops,
                                      threads=1)
            s[i], f[i] = ps[0], pf[0]
        return s, f

    res, fails = distributed.sharded_hafnian(nh, partials_fn, dist, rank, world, loops=loops)
    q.put((rank, res, fails))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,loops", [(2, 16, False), (3, 14, True)])
def test_sharded_gather_bit_identical(world, n, loops):
    from oracle import oracle as O
    from paper_1805_12498_b200 import workloads

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, loops, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    A = workloads.cfg2(n=n) if loops else workloads.cfg0(n=n)
    ref, rf = O.hafnian(A, 1, include_loops=loops)
    for rank, res, fails in out:
        assert fails == 0
        assert res == ref, (rank, res, ref)


def _bench_worker(rank, world, port, q):
    """bench.py's N>1 step orchestration with the device call mocked by the oracle: the
    rank's LPT shard of the fixed ranges -> its partials in a padded complex tensor ->
    bench.gather_shards (the all-gather) -> bench.assemble (range order + fixed tree);
    bench.max_over_ranks for the timing."""
    import torch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from oracle import oracle as O
    from paper_1805_12498_b200 import costmodel, workloads
    from paper_1805_12498_b200.engine import _prepare

    A = workloads.cfg0(n=18)
    at, dg, nh = _prepare(A, False)
    nr = min((1 << nh) - 1, bench.N_RANGES)
    shards = costmodel.lpt_shards(costmodel.range_costs(nh, nr), world)
    width = max(len(s) for s in shards)
    bounds = costmodel.range_bounds(nh, nr)
    local = torch.zeros(width, dtype=torch.complex128)
    for i, r in enumerate(shards[rank]):  # the mocked device call
        ps, _ = O.sum_mask_range(at, dg, nh, *bounds[r], 1, backend=1, threads=1)
        local[i] = complex(ps[0])
    gathered = [torch.zeros(width, dtype=torch.complex128) for _ in shards]
    bench.gather_shards(local, gathered, dist)
    res = bench.assemble(shards, gathered)
    t = bench.max_over_ranks([0.5 + rank, 3.0 - rank], dist, torch.device("cpu"))
    q.put((rank, res, t))
    dist.barrier()
    dist.destroy_process_group()


def test_bench_multirank_orchestration_gloo():
    from oracle import oracle as O
    from paper_1805_12498_b200 import workloads

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    ref, _ = O.hafnian(workloads.cfg0(n=18), 1)
    for rank, res, t in out:
        assert res == ref, (rank, res, ref)
        assert t == [1.5, 3.0]
