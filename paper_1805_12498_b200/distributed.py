"""Multi-GPU sharding of one hafnian's subset space (one process per GPU).

The reference's only "distributed" step is the paper's MPI sum of per-node
partial sums.  Here the 512 fixed mask ranges of the
deterministic contract (engine.N_RANGES) are the unit of sharding:

  * ranges are assigned to ranks by LPT on the closed-form cost model
    (costmodel.lpt_shards): max/mean rank load ~1.001 at 8 ranks, against
    1.34 for the reference's round-robin dealing (SURVEY.md finding 5);
  * every rank computes the Kahan partials of ITS ranges (no data-path
    collective: the terms never leave the GPU that computed them);
  * the partials are exchanged with one all-gather and every rank scatters
    them back into range order, so the fixed-tree result is bit-identical for
    any world size (the reference's deterministic contract, extended from
    threads to GPUs).

`partials_fn(ranges) -> (c128[len], int64[len])` computes a shard's partials;
on GPUs it is kernels.sum_range_list, in the CPU tests the oracle.
"""

from __future__ import annotations

import numpy as np

from . import costmodel
from .engine import N_RANGES, tree_reduce


def shard_plan(n_half: int, world: int, n_ranges: int | None = None, loops: bool = False):
    nr = n_ranges or min((1 << n_half) - 1, N_RANGES)
    costs = costmodel.range_costs(n_half, nr, loops)
    return nr, costmodel.lpt_shards(costs, world)


def gather_partials(local_sums, local_fails, shards, dist, rank: int):
    """All-gather every rank's shard partials (padded to the longest shard) and
    scatter them back into range order.  Works with any torch.distributed backend
    (NCCL tensors on the GPU ranks, gloo on CPU)."""
    import torch

    nr = sum(len(s) for s in shards)
    width = max(max(len(s) for s in shards), 1)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" \
        else torch.device("cpu")
    buf = torch.zeros(width, 3, dtype=torch.float64, device=dev)
    n = len(local_sums)
    if n:
        ls = np.asarray(local_sums, np.complex128)
        buf[:n, 0] = torch.from_numpy(ls.real.copy()).to(dev)
        buf[:n, 1] = torch.from_numpy(ls.imag.copy()).to(dev)
        buf[:n, 2] = torch.from_numpy(np.asarray(local_fails, np.float64)).to(dev)
    out = [torch.zeros_like(buf) for _ in shards]
    dist.all_gather(out, buf)
    sums = np.zeros(nr, np.complex128)
    fails = np.zeros(nr, np.int64)
    for r, s in enumerate(shards):
        if not s:
            continue
        o = out[r].cpu().numpy()[: len(s)]
        sums[s] = o[:, 0] + 1j * o[:, 1]
        fails[s] = o[:, 2].astype(np.int64)
    return sums, fails


def sharded_hafnian(n_half: int, partials_fn, dist, rank: int, world: int, loops: bool = False):
    """One hafnian over `world` ranks: LPT shard -> local partials -> all-gather ->
    fixed tree.  Returns (result, fails) on every rank."""
    nr, shards = shard_plan(n_half, world, loops=loops)
    mine = shards[rank]
    if mine:
        s, f = partials_fn(np.asarray(mine, np.int32))
    else:
        s, f = np.zeros(0, np.complex128), np.zeros(0, np.int64)
    sums, fails = gather_partials(s, f, shards, dist, rank)
    return tree_reduce(sums), int(fails.max()) if len(fails) else 0
