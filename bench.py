#!/usr/bin/env python
"""Headline benchmark: subset-terms/s of an n=52 hafnian on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One STEP = one full n=52 hafnian (cfg4, seed 3): all 2^26-1 signed subset terms,
the 512 fixed-range Kahan partials and (N>1) their gather.  The subset space is
sharded over ranks by LPT on the cost model (costmodel.py), so the total work is
fixed as N grows ("scaling": "strong").  Rank 0 prints ONE JSON line.

  value       terms/s over the K timed steps, inputs resident in HBM, CUDA events on
              the launching stream, max over ranks; 256 MiB L2 flush between steps
  e2e         the same metric through the public API with host inputs (hafnian() at
              N=1; the per-rank range-list ABI + host gather at N>1), wall clock
  roofline    FP64 roofline of the subset-term kernels: algorithmic FLOP of the
              step's shard (SURVEY 8(d) model) / terms-phase event time, against the
              FP64 peak measured by a DFMA probe in the same run
  cpu_baseline  the C restatement of the reference (oracle/, bit-identical to it) on
              the host cores, on a seeded uniform sample of the same workload's masks

--impl reference times that CPU implementation of the path (all host threads) on
the same workload, metric and unit (rank 0 only; other ranks exit 0).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

N_DEFAULT, SEED_DEFAULT, N_RANGES = 52, 3, 512
METRIC = "subset-terms/sec (n=52 hafnian)"


def metric_name(n: int) -> str:
    return METRIC if n == N_DEFAULT else f"subset-terms/sec (n={n} hafnian)"
UNIT = "terms/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=N_DEFAULT)
    ap.add_argument("--seed", type=int, default=SEED_DEFAULT)
    ap.add_argument("--arith", choices=["fast", "mirror"], default="fast")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--parity-bits", type=int, default=20,
                    help="check FAST/MIRROR against the CPU oracle on masks [0, 2^bits) (0 = skip)")
    ap.add_argument("--exact-steps", type=int, default=3,
                    help="timed runs of the exact GF(p) mode on cfg3 (0 = skip)")
    ap.add_argument("--mirror-steps", type=int, default=1,
                    help="timed steps in bit-exact MIRROR arithmetic (0 = skip)")
    return ap.parse_args()


def workload(args):
    from paper_1805_12498_b200 import engine, workloads

    A = workloads.cfg4(args.seed, args.n)
    at, dg, nh = engine._prepare(A, False)
    return A, at, dg, nh


def config(args, world):
    return {
        "workload": f"cfg4: hafnian of a complex symmetric n={args.n} matrix (seed {args.seed}, "
                    f"Gaussian/sqrt(n)), all 2^{args.n // 2}-1 subset terms per step",
        "n": args.n,
        "backend": "charpoly",
        "arith": args.arith,
        "n_ranges": N_RANGES,
        "parallelism": f"subset-range shards x{world} (LPT over {N_RANGES} ranges)",
        "l2": "256 MiB L2 flush between timed steps (per-step term buffer > L2 too)",
    }


# ------------------------------------------------------------------ CPU legs
def cpu_sample_rate(at, dg, nh, seconds, threads, seed=7):
    """Oracle (C restatement of the reference, charpoly backend) on a seeded uniform
    sample of the workload's masks; returns (terms/s, sample description)."""
    from oracle import oracle as O

    rng = np.random.default_rng(seed)
    probe = rng.integers(1, 1 << nh, 256, dtype=np.uint64)
    t0 = time.perf_counter()
    O.terms(at, dg, nh, probe, backend=1, threads=threads)
    dt = max(time.perf_counter() - t0, 1e-3)
    count = int(max(256, min(5_000_000, 256 * seconds / dt)))
    masks = rng.integers(1, 1 << nh, count, dtype=np.uint64)
    t0 = time.perf_counter()
    O.terms(at, dg, nh, masks, backend=1, threads=threads)
    dt = time.perf_counter() - t0
    return count / dt, count, dt


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as O

    O.build()
    _, at, dg, nh = workload(args)
    threads = len(os.sched_getaffinity(0))
    per_step = max(2.0, args.cpu_seconds / 2)
    rates = []
    desc = None
    for k in range(args.warmup + args.steps):
        r, count, dt = cpu_sample_rate(at, dg, nh, per_step, threads, seed=100 + k)
        if k >= args.warmup:
            rates.append(r)
            desc = f"{count} uniform random masks of the n={args.n} problem per step ({dt:.1f} s)"
    value = statistics.median(rates)
    print(json.dumps({
        "impl": "reference", "metric": metric_name(args.n), "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * ((1 << nh) - 1) / value, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64 (complex128)",
        "data": "synthetic (seeded, SURVEY.md Appendix A)", "config": config(args, 1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": desc + "; oracle/hafnian_oracle.c, bit-identical restatement "
                                          "of hafnium.kernels._numba (charpoly backend)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ GPU leg
def run_ours(args):
    import torch

    from paper_1805_12498_b200 import _lib, costmodel, engine, kernels

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = _lib.load(require_device=True)
    arith = kernels.ARITH_MODES[args.arith]
    A, at, dg, nh = workload(args)
    nterms = (1 << nh) - 1
    costs = costmodel.range_costs(nh, N_RANGES)
    shards = costmodel.lpt_shards(costs, world)
    mine = np.ascontiguousarray(shards[rank], dtype=np.int32)
    bounds = costmodel.range_bounds(nh, N_RANGES)
    my_flops = sum(costmodel.flops_of_range(*bounds[r], nh) for r in mine)

    peak_tf = ctypes.c_double()
    peak_ms = ctypes.c_double()
    _lib.check(lib.hafb_fp64_peak(local, ctypes.byref(peak_tf), ctypes.byref(peak_ms)))

    dev = torch.device("cuda", local)
    d_at = torch.from_numpy(at).to(dev)
    d_dg = torch.from_numpy(dg).to(dev)
    cnt = int(mine.size)
    width = max(max(len(s) for s in shards), 1)  # all-gather needs equal sizes
    d_part = torch.zeros(width, dtype=torch.complex128, device=dev)
    d_fail = torch.zeros(width, dtype=torch.int64, device=dev)
    ws_bytes = int(lib.hafb_range_list_workspace_bytes(nh, N_RANGES, cnt))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    gathered = [torch.zeros(width, dtype=torch.complex128, device=dev) for _ in shards]

    def step(ev_terms=None):
        if cnt:
            _lib.check(lib.hafb_sum_range_list_async(
                ctypes.c_void_p(d_at.data_ptr()), ctypes.c_void_p(d_dg.data_ptr()), nh, N_RANGES,
                _lib.i32ptr(mine), cnt, 1, 0, kernels.SWEEP_CAP_MULT, arith,
                ctypes.c_void_p(ws.data_ptr()), ws_bytes, ctypes.c_void_p(d_part.data_ptr()),
                ctypes.c_void_p(d_fail.data_ptr()), ctypes.c_void_p(stream.cuda_stream),
                ctypes.c_void_p(ev_terms.cuda_event if ev_terms is not None else 0)))
        if dist is not None:  # the exchange: per-rank range partials -> every rank
            dist.all_gather([torch.view_as_real(g) for g in gathered], torch.view_as_real(d_part))

    def assemble():
        parts = np.zeros(N_RANGES, np.complex128)
        for r, s in enumerate(shards):
            if s:
                parts[s] = gathered[r].cpu().numpy()[: len(s)] if dist is not None else \
                    d_part.cpu().numpy()[: len(s)]
        return engine.tree_reduce(parts)

    for _ in range(args.warmup):
        step()
        flush.zero_()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    lib.hafb_launch_count(1)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
            torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for _, et, _ in evs:  # materialise the lazily created events before the ABI records them
        et.record(stream)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        e0, et, e1 = evs[k]
        e0.record(stream)
        step(et)
        e1.record(stream)
        flush.zero_()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    launches = int(lib.hafb_launch_count(1))
    clk = clocks.stop()
    step_ms = [e0.elapsed_time(e1) for e0, _, e1 in evs]
    terms_ms = [e0.elapsed_time(et) for e0, et, _ in evs]
    total_s = sum(step_ms) / 1e3
    terms_s = sum(terms_ms) / 1e3
    if dist is not None:
        t = torch.tensor([total_s, terms_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_max, _ = t.tolist()
    else:
        total_max = total_s
    result = assemble()
    value = args.steps * nterms / total_max
    achieved = my_flops / (terms_s / args.steps) / 1e12

    # e2e: host inputs through the public API, wall clock (incl. H2D / D2H every step)
    e2e_times = []
    h2d = (at.nbytes + dg.nbytes)
    d2h = 16 * max(cnt, 1) + 8 * max(cnt, 1)
    for k in range(args.warmup + args.steps):
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        if world == 1:
            r_e2e = engine.hafnian(A, backend="charpoly", arith=args.arith)
        else:
            from paper_1805_12498_b200 import distributed

            r_e2e, _ = distributed.sharded_hafnian(
                nh, lambda rl: kernels.sum_range_list(at, dg, nh, N_RANGES, rl, 1, False,
                                                      arith=args.arith, device=local),
                dist, rank, world)
        dt = time.perf_counter() - t0
        if dist is not None:
            t = torch.tensor([dt], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        if k >= args.warmup:
            e2e_times.append(dt)
    e2e_value = nterms / statistics.median(e2e_times)

    # bit-exact MIRROR arithmetic on the same step (reported beside the headline)
    mirror = None
    if args.mirror_steps > 0:
        m_ms = []
        for _ in range(args.mirror_steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if cnt:
                _lib.check(lib.hafb_sum_range_list_async(
                    ctypes.c_void_p(d_at.data_ptr()), ctypes.c_void_p(d_dg.data_ptr()), nh,
                    N_RANGES, _lib.i32ptr(mine), cnt, 1, 0, kernels.SWEEP_CAP_MULT,
                    kernels.ARITH_MODES["mirror"], ctypes.c_void_p(ws.data_ptr()), ws_bytes,
                    ctypes.c_void_p(d_part.data_ptr()), ctypes.c_void_p(d_fail.data_ptr()),
                    ctypes.c_void_p(stream.cuda_stream), ctypes.c_void_p(0)))
            if dist is not None:
                dist.all_gather([torch.view_as_real(g) for g in gathered], torch.view_as_real(d_part))
            e1.record(stream)
            torch.cuda.synchronize()
            m_ms.append(e0.elapsed_time(e1))
        m_s = max(m_ms) / 1e3
        if dist is not None:
            t = torch.tensor([m_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            m_s = float(t.item())
        mres = assemble()
        mirror = {"value": nterms / m_s, "unit": UNIT, "sec_per_hafnian": m_s,
                  "steps": args.mirror_steps, "result": [mres.real, mres.imag],
                  "rel_diff_fast_vs_mirror": abs(result - mres) / abs(mres) if mres else None,
                  "note": "arith=mirror reproduces the reference's IEEE operation sequence; its "
                          "terms and partials are bit-identical to hafnium's numba kernels "
                          "(tests/test_gpu_parity.py)"}

    # exact GF(p)+CRT mode on cfg3 (integer matching count, beyond float precision)
    exact_line = None
    if rank == 0 and args.exact_steps > 0:
        from paper_1805_12498_b200 import exact as X, workloads

        a3 = workloads.cfg3()
        X.hafnian_exact(a3)  # warm-up
        ts = []
        for _ in range(args.exact_steps):
            t0 = time.perf_counter()
            cnt3 = X.hafnian_exact(a3)
            ts.append(time.perf_counter() - t0)
        t3 = statistics.median(ts)
        exact_line = {"workload": "cfg3: perfect matchings of an ER(0.5) n=40 graph (seed 2)",
                      "value": (2**20 - 1) / t3, "unit": "subset-terms/s (3 primes, host prep included)",
                      "sec": t3, "result": str(cnt3),
                      "matches_known_answer": cnt3 == 308544357990268074}

    # parity at full size (north star: identical contiguous subset range at n >= 48):
    # FAST and MIRROR against the CPU oracle (bit-pinned to the reference) on [0, 2^20)
    parity = None
    if rank == 0 and args.parity_bits > 0:
        from oracle import oracle as O

        O.build()
        hi = 1 << min(args.parity_bits, nh)
        masks = np.arange(1, hi, dtype=np.uint64)
        thr = len(os.sched_getaffinity(0))
        t_orc = O.terms(at, dg, nh, masks, backend=1, threads=thr)[0]
        t_fast, _ = kernels.terms(at, dg, nh, masks, 1, False, arith="fast", device=local)
        t_mir, _ = kernels.terms(at, dg, nh, masks, 1, False, arith="mirror", device=local)
        n_ch = 8
        r_orc = O.tree_reduce(O.sum_mask_range(at, dg, nh, 0, hi, n_ch, 1, False)[0])
        r_fast = engine.tree_reduce(kernels.sum_mask_range(at, dg, nh, 0, hi, n_ch, 1, False,
                                                               arith="fast", device=local)[0])
        r_mir = engine.tree_reduce(kernels.sum_mask_range(at, dg, nh, 0, hi, n_ch, 1, False,
                                                              arith="mirror", device=local)[0])
        abs_sum = float(np.abs(t_orc).sum())
        den = np.maximum(np.abs(t_orc), 1e-300)
        parity = {
            "range": f"masks [0, 2^{min(args.parity_bits, nh)}) of the n={args.n} workload, "
                     f"{n_ch} Kahan chunks + fixed tree (SURVEY.md 8(c) harness)",
            "oracle": "oracle/hafnian_oracle.c (bit-identical to hafnium.kernels._numba on the "
                      "golden fixtures), charpoly backend",
            "tolerance": {"rel": 1e-10, "abs_sum_normalised": 1e-15,
                          "rule": "FAST passes if |r-ref| <= max(1e-10 |ref|, 1e-15 sum|t|); "
                                  "MIRROR must be bit-identical"},
            "fast_rel_err": abs(r_fast - r_orc) / abs(r_orc),
            "fast_abs_sum_normalised_err": abs(r_fast - r_orc) / abs_sum,
            "fast_max_term_rel_err": float((np.abs(t_fast - t_orc) / den).max()),
            "mirror_bit_identical_result": bool(r_mir == r_orc),
            "mirror_bit_identical_terms": int((np.ascontiguousarray(t_mir).view(np.uint64).reshape(-1, 2)
                                               == np.ascontiguousarray(t_orc).view(np.uint64).reshape(-1, 2))
                                              .all(axis=1).sum()),
            "terms": int(masks.size),
            "cond_abs_sum_over_result": abs_sum / abs(r_orc),
        }
        parity["pass"] = (parity["fast_rel_err"] <= 1e-10
                          or parity["fast_abs_sum_normalised_err"] <= 1e-15) \
            and parity["mirror_bit_identical_result"]

    cpu = None
    if rank == 0 and world == 1:
        from oracle import oracle as O

        O.build()
        threads = len(os.sched_getaffinity(0))
        rate, count, dt = cpu_sample_rate(at, dg, nh, args.cpu_seconds, threads)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{count} uniform random masks of the n={args.n} problem ({dt:.1f} s); "
                         "oracle/hafnian_oracle.c, bit-identical restatement of "
                         "hafnium.kernels._numba (charpoly backend)"}

    traffic = None
    tpath = os.path.join(REPO, "profiles", "roofline_traffic.json")
    if os.path.exists(tpath):
        try:
            # measured DRAM bytes per term of the term kernels (profiles/roofline_traffic.json),
            # per launch-set of one step
            traffic = json.load(open(tpath)).get("bytes_per_term") * nterms
        except (ValueError, OSError):
            traffic = None

    if rank == 0:
        line = {
            "metric": metric_name(args.n), "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64 (complex128)", "data": "synthetic (seeded, SURVEY.md Appendix A)",
            "config": config(args, world),
            "sec_per_hafnian": total_max / args.steps,
            "result": [result.real, result.imag],
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak_tf.value,
                         "unit": "TFLOP/s", "frac": achieved / peak_tf.value, "traffic": traffic,
                         "peak_source": "DFMA probe measured in this run (hafb_fp64_peak); "
                                        "MEASURED_PEAKS.json has no FP64 entry",
                         "flop_model": "SURVEY.md 8(d) CMA model, 8 FLOP per complex MAC"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clk,
        }
        if mirror is not None:
            line["mirror"] = mirror
        if exact_line is not None:
            line["exact"] = exact_line
        if parity is not None:
            line["parity"] = parity
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
