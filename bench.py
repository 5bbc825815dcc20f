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
              FP64 peak measured by a DFMA probe in the same run (and, as frac_nominal,
              against the 37.2 TF/s datasheet figure 148 SMs x 64 DFMA/clk x 2 x 1.965 GHz)
  configs     every BASELINE config (cfg0..cfg4 incl. the 4096-matrix batch, the loop
              hafnian, n=56 and seed 4): terms/s, s/hafnian, roofline fractions, accuracy
              against the extended-precision referee, and the reference's CPU time
  spectral    the reference's default backend (spectral: Hessenberg + shifted QR) on the
              identical range [0, 2^20): FAST spectral, bit-exact MIRROR spectral (checked
              against the C oracle), the unmodified reference and the C port on host cores
  cpu_baseline  the UNMODIFIED reference (hafnium 0.1.0 numba kernels, installed in
              baseline/_ref) on all host cores, on a seeded uniform sample of the same
              workload's masks; the C port of it (oracle/) beside it

--impl reference times the reference's own CPU implementation of the path (numba,
all host threads; the C port if numba or baseline/_ref is unavailable) on the same
workload, metric and unit: each step is a bounded uniform sample of the n=52
problem's masks (rank 0 only; other ranks exit 0).
"""

from __future__ import annotations

import argparse
import ctypes
import json
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
UNIT = "terms/s"
NOMINAL_FP64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # datasheet-style DFMA peak at max clock


def metric_name(n: int) -> str:
    return METRIC if n == N_DEFAULT else f"subset-terms/sec (n={n} hafnian)"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=N_DEFAULT)
    ap.add_argument("--seed", type=int, default=SEED_DEFAULT)
    ap.add_argument("--arith", choices=["fast", "mirror"], default="fast")
    ap.add_argument("--spectral-bits", type=int, default=20,
                    help="spectral-backend leg on masks [0, 2^bits) (0 = skip)")
    ap.add_argument("--cpu-seconds", type=float, default=8.0,
                    help="CPU budget of the headline cpu_baseline sample")
    ap.add_argument("--ref-step-seconds", type=float, default=1.0,
                    help="--impl reference: CPU seconds per step (a bounded sample)")
    ap.add_argument("--parity-bits", type=int, default=20,
                    help="check FAST/MIRROR against the CPU oracle on masks [0, 2^bits) (0 = skip)")
    ap.add_argument("--exact-steps", type=int, default=3,
                    help="timed runs of the exact GF(p) mode on cfg3 (0 = skip)")
    ap.add_argument("--mirror-steps", type=int, default=1,
                    help="timed steps in bit-exact MIRROR arithmetic (0 = skip)")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config legs")
    ap.add_argument("--no-proxy", action="store_true", help="skip the multi-GPU shard proxy")
    return ap.parse_args(argv)


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


# ------------------------------------------------------------------ CPU: the reference itself
class NumbaReference:
    """The unmodified reference (hafnium 0.1.0 from baseline/_ref, numba kernels) driven by
    the SURVEY.md 8(c) harness: its own ``kernels._numba.subset_term`` over an array of
    masks in a numba prange loop (the reference has no range API; its public
    ``hafnium.hafnian`` runs the same subset_term per mask inside sum_subsets_det)."""

    def __init__(self, threads):
        ref = os.path.join(REPO, "baseline", "_ref")
        if not os.path.isdir(os.path.join(ref, "hafnium")):
            raise ImportError("baseline/_ref/hafnium is not installed")
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/hafb_numba_cache")
        if ref not in sys.path:
            sys.path.insert(0, ref)
        import numba
        from hafnium.kernels import _numba as nb

        numba.set_num_threads(threads)
        self.threads = threads
        sub = nb.subset_term
        cap = nb.SWEEP_CAP_MULT

        @numba.njit(parallel=True)
        def run(atilde, diag, n_half, masks, backend, loops):
            out = np.zeros(masks.size, np.complex128)
            for q in numba.prange(masks.size):
                t, s = sub(atilde, diag, masks[q], n_half, backend, loops, cap)
                out[q] = t
            return out

        self._run = run

    def terms(self, at, dg, nh, masks, backend, loops=False):
        return self._run(at, dg, nh, np.ascontiguousarray(masks, np.int64), backend, bool(loops))

    def rate(self, at, dg, nh, backend, seconds, loops=False, seed=7, all_masks=False):
        """terms/s on a seeded uniform sample of masks sized to ~`seconds` (every mask of
        the problem when all_masks and it fits).  Returns (rate, count, dt)."""
        rng = np.random.default_rng(seed)
        total = (1 << nh) - 1
        self.terms(at, dg, nh, rng.integers(1, total + 1, 64), backend, loops)  # JIT
        probe = rng.integers(1, total + 1, 256 * self.threads)
        t0 = time.perf_counter()
        self.terms(at, dg, nh, probe, backend, loops)
        dt = max(time.perf_counter() - t0, 1e-4)
        count = int(max(256, min(4_000_000, probe.size * seconds / dt)))
        if all_masks and count >= total:
            masks = np.arange(1, total + 1)
        else:
            masks = rng.integers(1, total + 1, count)
        t0 = time.perf_counter()
        self.terms(at, dg, nh, masks, backend, loops)
        dt = time.perf_counter() - t0
        return masks.size / dt, int(masks.size), dt


def port_rate(at, dg, nh, seconds, threads, seed=7, loops=False):
    """The C restatement of the reference (oracle/, bit-identical to it, charpoly
    backend) on a seeded uniform sample of the workload's masks."""
    from oracle import oracle as O

    O.build()
    rng = np.random.default_rng(seed)
    probe = rng.integers(1, 1 << nh, 256, dtype=np.uint64)
    t0 = time.perf_counter()
    O.terms(at, dg, nh, probe, backend=1, include_loops=loops, threads=threads)
    dt = max(time.perf_counter() - t0, 1e-3)
    count = int(max(256, min(5_000_000, 256 * seconds / dt)))
    masks = rng.integers(1, 1 << nh, count, dtype=np.uint64)
    t0 = time.perf_counter()
    O.terms(at, dg, nh, masks, backend=1, include_loops=loops, threads=threads)
    dt = time.perf_counter() - t0
    return count / dt, count, dt


def run_spectral(at, dg, nh, device, args, cref, threads, ref_cache):
    """backend='spectral' (the reference's default) on masks [0, 2^bits) of the workload:
    FAST and MIRROR through the range ABI (host inputs, partials back; best of 2 after a
    warm-up), the reference (numba) and the C port on a uniform sample of the same range,
    MIRROR checked bit for bit against the C oracle and FAST against the referee."""
    from oracle import oracle as O
    from paper_1805_12498_b200 import engine, kernels

    bits = min(args.spectral_bits, nh)
    hi = 1 << bits
    nterms = hi - 1
    out = {"range": f"masks [0, 2^{bits}) of the n={args.n} workload (seed {args.seed}), 512 Kahan "
                    f"chunks + fixed tree", "terms": nterms}
    res = {}
    for arith in ("fast", "mirror"):
        kernels.sum_mask_range(at, dg, nh, 0, min(hi, 1 << 12), 512, 0, False, arith=arith, device=device)
        ts = []
        for _ in range(2):
            t0 = time.perf_counter()
            sums, fails = kernels.sum_mask_range(at, dg, nh, 0, hi, 512, 0, False, arith=arith, device=device)
            ts.append(time.perf_counter() - t0)
        r = engine.tree_reduce(sums)
        res[arith] = r
        out[arith] = {"value": nterms / min(ts), "unit": UNIT, "sec": min(ts), "result": [r.real, r.imag],
                      "fails": int(fails.max())}
    O.build()
    r_orc = O.tree_reduce(O.sum_mask_range(at, dg, nh, 0, hi, 512, 0, False)[0])
    out["mirror"]["bit_identical_to_oracle"] = bool(res["mirror"] == r_orc)
    key = f"range_n{args.n}s{args.seed}"
    if bits == 20 and key in ref_cache:
        out["fast"]["accuracy"] = _score(res["fast"], ref_cache, key)
        out["mirror"]["accuracy"] = _score(res["mirror"], ref_cache, key)
    rng = np.random.default_rng(11)
    masks = rng.integers(1, hi, 20000, dtype=np.uint64)
    t0 = time.perf_counter()
    O.terms(at, dg, nh, masks, backend=0, threads=threads)
    dt = time.perf_counter() - t0
    out["cpu_port"] = {"value": masks.size / dt, "unit": UNIT, "cores": threads, "kind": "port",
                       "sample": f"{masks.size} uniform masks of the range ({dt:.2f} s), oracle/"
                                 f"hafnian_oracle.c spectral"}
    if cref is not None:
        cref.terms(at, dg, nh, masks[:64].astype(np.int64), 0)  # JIT
        t0 = time.perf_counter()
        cref.terms(at, dg, nh, masks.astype(np.int64), 0)
        dt = time.perf_counter() - t0
        out["cpu_reference"] = {"value": masks.size / dt, "unit": UNIT, "cores": threads,
                                "kind": "reference",
                                "sample": f"{masks.size} uniform masks of the range ({dt:.2f} s), the "
                                          f"unmodified reference (numba, backend=0)"}
        out["speedup_fast_vs_reference"] = out["fast"]["value"] / out["cpu_reference"]["value"]
    out["speedup_fast_vs_port"] = out["fast"]["value"] / out["cpu_port"]["value"]
    return out


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    _, at, dg, nh = workload(args)
    threads = len(os.sched_getaffinity(0))
    nterms = (1 << nh) - 1
    try:
        ref = NumbaReference(threads)
        kind, what = "reference", ("the unmodified reference (baseline/_ref hafnium 0.1.0, numba "
                                   "kernels, charpoly backend) via its kernels._numba.subset_term")

        def sample(seconds, seed):
            return ref.rate(at, dg, nh, 1, seconds, seed=seed)
    except ImportError as e:
        kind, what = "port", (f"oracle/hafnian_oracle.c, the bit-identical C restatement of "
                              f"hafnium.kernels._numba (charpoly backend; numba reference "
                              f"unavailable: {e})")

        def sample(seconds, seed):
            return port_rate(at, dg, nh, seconds, threads, seed=seed)

    rates, step_s, desc = [], [], None
    for k in range(args.warmup + args.steps):
        r, count, dt = sample(args.ref_step_seconds, 100 + k)
        if k >= args.warmup:
            rates.append(r)
            step_s.append(dt)
            desc = (f"{count} uniform random masks of the n={args.n} problem per step "
                    f"({dt:.2f} s, {threads} threads); {what}")
    value = statistics.median(rates)
    line = {
        "impl": "reference", "metric": metric_name(args.n), "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.median(step_s), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64 (complex128)",
        "data": "synthetic (seeded, SURVEY.md Appendix A)", "config": config(args, 1),
        "step": "one bounded uniform sample of the workload's subset masks (the full hafnian "
                "would take sec_per_hafnian_extrapolated)",
        "sec_per_hafnian_extrapolated": nterms / value,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": desc, "cpu": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if kind == "reference":  # the reference's default backend, for the record
        r0, c0, d0 = ref.rate(at, dg, nh, 0, max(0.5, args.ref_step_seconds / 2), seed=99)
        line["spectral"] = {"value": r0, "unit": UNIT, "sample": f"{c0} masks ({d0:.2f} s)",
                            "note": "backend='spectral' (the reference default): Hessenberg + "
                                    "shifted QR per subset"}
    print(json.dumps(line), flush=True)


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


# ------------------------------------------------------------------ multi-rank plumbing
def max_over_ranks(values, dist, device):
    """Element-wise max of a few floats over all ranks (works for nccl and gloo)."""
    if dist is None:
        return list(values)
    import torch

    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def gather_shards(local, gathered, dist):
    """The step's only exchange: every rank's range partials (a complex tensor padded to
    the longest shard) to every rank."""
    import torch

    if dist is not None:
        dist.all_gather([torch.view_as_real(g) for g in gathered], torch.view_as_real(local))


def assemble(shards, gathered, local=None):
    """Scatter the gathered shard partials back into range order and apply the fixed tree
    (bit-identical to the single-device result for every world size)."""
    from paper_1805_12498_b200 import engine

    parts = np.zeros(sum(len(s) for s in shards), np.complex128)
    for r, s in enumerate(shards):
        if s:
            src = gathered[r] if local is None else local
            parts[s] = src.cpu().numpy()[: len(s)]
    return engine.tree_reduce(parts)


# ------------------------------------------------------------------ device problem
class DeviceProblem:
    """One prepared problem resident in HBM and its range-list launch (the
    hafb_sum_range_list_async ABI): `launch(ranges, arith)` enqueues the subset-term
    kernels and the Kahan range reduction on `stream`."""

    def __init__(self, lib, at, dg, nh, loops, device, stream, max_ranges=None):
        import torch

        from paper_1805_12498_b200 import _lib

        self.lib, self._lib = lib, _lib
        self.nh, self.loops, self.stream = nh, bool(loops), stream
        self.n_ranges = min((1 << nh) - 1, N_RANGES)
        cnt = max_ranges or self.n_ranges
        self.d_at = torch.from_numpy(np.ascontiguousarray(at)).to(device)
        self.d_dg = torch.from_numpy(np.ascontiguousarray(dg)).to(device)
        self.d_part = torch.zeros(max(cnt, 1), dtype=torch.complex128, device=device)
        self.d_fail = torch.zeros(max(cnt, 1), dtype=torch.int64, device=device)
        self.ws_bytes = int(lib.hafb_range_list_workspace_bytes(nh, self.n_ranges, self.n_ranges))
        self.ws = torch.empty(max(self.ws_bytes, 1), dtype=torch.uint8, device=device)

    def launch(self, ranges, arith, ev_terms=None):
        from paper_1805_12498_b200 import kernels

        rl = np.ascontiguousarray(ranges, dtype=np.int32)
        if not rl.size:
            return
        self._lib.check(self.lib.hafb_sum_range_list_async(
            ctypes.c_void_p(self.d_at.data_ptr()), ctypes.c_void_p(self.d_dg.data_ptr()), self.nh,
            self.n_ranges, self._lib.i32ptr(rl), int(rl.size), 1, int(self.loops),
            kernels.SWEEP_CAP_MULT, kernels.ARITH_MODES[arith], ctypes.c_void_p(self.ws.data_ptr()),
            self.ws_bytes, ctypes.c_void_p(self.d_part.data_ptr()),
            ctypes.c_void_p(self.d_fail.data_ptr()), ctypes.c_void_p(self.stream.cuda_stream),
            ctypes.c_void_p(ev_terms.cuda_event if ev_terms is not None else 0)))

    def time_ms(self, ranges, arith, reps=1, warm=True):
        """Median event time (ms) of `reps` launches (after one untimed launch if warm)."""
        import torch

        ts = []
        if warm:
            self.launch(ranges, arith)
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(self.stream)
            self.launch(ranges, arith)
            e1.record(self.stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    def result(self):
        from paper_1805_12498_b200 import engine

        return engine.tree_reduce(self.d_part.cpu().numpy()[: self.n_ranges])


def _wall(fn, reps):
    ts, out = [], None
    fn()
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts), out


# ------------------------------------------------------------------ per-config legs
def _referee():
    """Extended-precision referee values (tests/golden, generated by oracle/referee.c)."""
    g = os.path.join(REPO, "tests", "golden")
    out = {}
    try:
        z = np.load(os.path.join(g, "referee.npz"))
        for k in z.files:
            grp, field = k.split("/", 1)
            out.setdefault(grp, {})[field] = z[k]
        if os.path.exists(os.path.join(g, "referee_full52.npz")):
            f = np.load(os.path.join(g, "referee_full52.npz"))
            out["full_n52s3"] = {k: f[k] for k in f.files}
        if os.path.exists(os.path.join(g, "referee_batch.npz")):
            out["batch"] = dict(np.load(os.path.join(g, "referee_batch.npz")))
        ranges = np.load(os.path.join(g, "ranges.npz"))
        r52 = np.load(os.path.join(g, "range_n52.npz"))
        out["_reference_results"] = {k.split("/")[0]: complex(ranges[k]) for k in ranges.files
                                     if k.endswith("/result_b1")}
        out["_reference_results"].update({f"range_{k.split('/')[0]}": complex(r52[k])
                                          for k in r52.files if k.endswith("/result_b1")})
        bpath = os.path.join(g, "batch_cfg1.npz")
        if os.path.exists(bpath):
            out["_batch_reference"] = dict(np.load(bpath))
    except (OSError, ValueError):
        pass
    return out


def _score(x, ref, key):
    from paper_1805_12498_b200 import accuracy

    if key not in ref:
        return None
    hi, lo, sa = complex(ref[key]["hi"]), complex(ref[key]["lo"]), float(ref[key]["abs_sum"])
    return {"rel_err_vs_referee": accuracy.error(x, hi, lo) / abs(hi),
            "within_bound": bool(accuracy.within(x, hi, lo, sa)),
            "cond": sa / abs(hi)}


def _roof(flop, seconds, peak):
    tf = flop / seconds / 1e12
    return {"tflops": tf, "frac_probe": tf / peak, "frac_nominal": tf / NOMINAL_FP64_TFLOPS}


def run_configs(lib, device, stream, peak, cref, threads, ref_cache):
    """Every BASELINE config on one GPU: FAST device time (range-list ABI, events), FAST
    and MIRROR end to end through the public API, accuracy against the referee, and the
    reference's own CPU rate (both backends) on the box's cores."""
    from paper_1805_12498_b200 import costmodel, engine, workloads

    legs = {}
    cases = [
        ("cfg0", workloads.cfg0(), False, "single hafnian n=20, seed 0", 20),
        ("cfg2", workloads.cfg2(), True, "loop hafnian n=32, seed 1", 10),
        ("cfg3", workloads.cfg3(), False, "ER(0.5) perfect-matching count n=40, seed 2 (float)", 5),
        ("cfg4_n52s4", workloads.cfg4(4, 52), False, "hafnian n=52, seed 4", 1),
        ("cfg4_n56s4", workloads.cfg4(4, 56), False, "hafnian n=56, seed 4 (timing)", 1),
    ]
    for name, A, loops, desc, reps in cases:
        at, dg, nh = engine._prepare(A, loops)
        nterms = (1 << nh) - 1
        flop = costmodel.flops_total(nh, loops)
        prob = DeviceProblem(lib, at, dg, nh, loops, device, stream)
        all_r = list(range(prob.n_ranges))
        big = nh >= 26
        dev_s = prob.time_ms(all_r, "fast", reps, warm=not big) / 1e3
        fres = prob.result()
        f = engine.loop_hafnian if loops else engine.hafnian
        leg = {"workload": desc, "n": 2 * nh, "terms": nterms, "flop": flop,
               "fast": {"sec_per_hafnian": dev_s, "value": nterms / dev_s, "unit": UNIT,
                        **_roof(flop, dev_s, peak), "result": [fres.real, fres.imag]}}
        fast_api = fres
        if nh < 28:  # end to end through the public API (n=56: device time only)
            e2e_s, fast_api = _wall(lambda: f(A, backend="charpoly", arith="fast"),
                                    max(1, min(reps, 5)))
            leg["fast"].update({"e2e_sec": e2e_s, "e2e_value": nterms / e2e_s,
                                "public_api_equals_device_abi": bool(fast_api == fres)})
        else:
            e2e_s = dev_s
        if nh <= 26:
            m_s, mres = _wall(lambda: f(A, backend="charpoly", arith="mirror"), 1)
            leg["mirror"] = {"e2e_sec": m_s, "e2e_value": nterms / m_s,
                             "result": [mres.real, mres.imag]}
            ref_val = ref_cache.get("_reference_results", {}).get(name)
            if ref_val is not None:
                leg["mirror"]["bit_identical_to_reference"] = bool(mres == ref_val)
        acc = {}
        key = {"cfg4_n52s4": None, "cfg4_n56s4": None}.get(name, name)
        if key:
            acc["fast"] = _score(fast_api, ref_cache, key)
            if "mirror" in leg:
                acc["mirror_eq_reference"] = _score(complex(*leg["mirror"]["result"]), ref_cache, key)
        if name == "cfg3":
            exact = 308544357990268074
            acc["fast_rel_err_vs_exact_count"] = abs(fast_api.real - exact) / exact
            acc["reference_rel_err_vs_exact_count"] = abs(
                ref_cache.get("_reference_results", {}).get("cfg3", complex("nan")).real - exact) / exact
        if acc:
            leg["accuracy"] = acc
        if cref is not None:
            c1, n1, d1 = cref.rate(at, dg, nh, 1, 0.6, loops=loops, seed=11, all_masks=True)
            c0, n0, d0 = cref.rate(at, dg, nh, 0, 0.6, loops=loops, seed=12, all_masks=True)
            leg["cpu_reference"] = {
                "cores": threads, "kind": "reference",
                "charpoly": {"value": c1, "unit": UNIT, "sec_per_hafnian": nterms / c1,
                             "sample": f"{n1} masks ({d1:.2f} s)",
                             "extrapolated": n1 < nterms},
                "spectral": {"value": c0, "unit": UNIT, "sec_per_hafnian": nterms / c0,
                             "sample": f"{n0} masks ({d0:.2f} s)",
                             "extrapolated": n0 < nterms},
                "speedup_fast_e2e_vs_charpoly": (nterms / e2e_s) / c1}
        legs[name] = leg
        del prob
    legs["cfg1"] = run_batch_leg(peak, cref, threads, ref_cache)
    return legs


def run_batch_leg(peak, cref, threads, ref_cache):
    """cfg1: the 4096-matrix GBS-like batch through hafnian_batch (host inputs, end to end;
    the reference has no batch API and loops hafnian())."""
    from paper_1805_12498_b200 import accuracy, costmodel, engine, workloads

    count, nh = 4096, 12
    As = np.array([workloads.cfg1(s) for s in range(count)])
    nterms = count * ((1 << nh) - 1)
    flop = count * costmodel.flops_total(nh)
    f_s, fres = _wall(lambda: engine.hafnian_batch(As, backend="charpoly", arith="fast"), 3)
    m_s, mres = _wall(lambda: engine.hafnian_batch(As, backend="charpoly", arith="mirror"), 1)
    leg = {"workload": "batch of 4096 GBS-like hafnians n=24, seeds 0..4095", "n": 24,
           "terms": nterms, "flop": flop,
           "fast": {"e2e_sec": f_s, "e2e_value": nterms / f_s, "unit": UNIT,
                    "sec_per_hafnian": f_s / count, **_roof(flop, f_s, peak),
                    "h2d_bytes": int(As.nbytes), "note": "end to end incl. H2D of the batch"},
           "mirror": {"e2e_sec": m_s, "e2e_value": nterms / m_s}}
    B, G = ref_cache.get("batch"), ref_cache.get("_batch_reference")
    if B is not None and G is not None:
        hi, lo, sa = B["hi"], B["lo"], B["abs_sum"]
        ef = np.abs((fres - hi) - lo) / np.abs(hi)
        er = np.abs((G["result_b1"] - hi) - lo) / np.abs(hi)
        bound = np.maximum(accuracy.REL * np.abs(hi), accuracy.ABS_SUM * sa)
        leg["accuracy"] = {
            "mirror_bit_identical_to_reference": int(np.sum(mres == G["result_b1"])),
            "fast_within_bound": int(np.sum(np.abs((fres - hi) - lo) <= bound)),
            "fast_rel_err_q50_q99_max": [float(x) for x in np.quantile(ef, [0.5, 0.99, 1.0])],
            "reference_rel_err_q50_q99_max": [float(x) for x in np.quantile(er, [0.5, 0.99, 1.0])],
            "fast_above_1e-10": int(np.sum(ef > 1e-10)),
            "reference_above_1e-10": int(np.sum(er > 1e-10))}
    if cref is not None:
        # the reference loops hafnian() over the batch: time it on a bounded prefix
        import hafnium

        sub = 48
        hafnium.hafnian(As[0], backend="charpoly", threads=threads)
        t0 = time.perf_counter()
        for a in As[:sub]:
            hafnium.hafnian(a, backend="charpoly", threads=threads)
        dt = time.perf_counter() - t0
        leg["cpu_reference"] = {"cores": threads, "kind": "reference",
                                "charpoly": {"value": sub * ((1 << nh) - 1) / dt, "unit": UNIT,
                                             "sec_per_batch": dt * count / sub, "extrapolated": True,
                                             "sample": f"hafnium.hafnian(threads={threads}) over the "
                                                       f"first {sub} matrices ({dt:.2f} s)"},
                                "speedup_fast_e2e_vs_charpoly": (dt * count / sub) / f_s}
    return leg


def run_proxy(lib, at, dg, nh, device, stream, full_s):
    """Multi-GPU readiness on one GPU: each rank's LPT shard of the n=52 step timed alone
    (the range-list path a rank runs); proxy efficiency at k ranks = full step time /
    (k x the slowest shard's time)."""
    from paper_1805_12498_b200 import costmodel

    prob = DeviceProblem(lib, at, dg, nh, False, device, stream)
    costs = costmodel.range_costs(nh, N_RANGES)
    out = {}
    for k in (2, 4, 8):
        shards = costmodel.lpt_shards(costs, k)
        ts = [prob.time_ms(s, "fast", 1) / 1e3 for s in shards]
        out[str(k)] = {"shard_sec": ts, "max_shard_sec": max(ts),
                       "proxy_efficiency": full_s / (k * max(ts)),
                       "cost_imbalance": costmodel.imbalance(costs, shards)}
    return out


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
    A, at, dg, nh = workload(args)
    nterms = (1 << nh) - 1
    costs = costmodel.range_costs(nh, N_RANGES)
    shards = costmodel.lpt_shards(costs, world)
    mine = shards[rank]
    bounds = costmodel.range_bounds(nh, N_RANGES)
    my_flops = sum(costmodel.flops_of_range(*bounds[r], nh) for r in mine)

    peak_tf = ctypes.c_double()
    peak_ms = ctypes.c_double()
    _lib.check(lib.hafb_fp64_peak(local, ctypes.byref(peak_tf), ctypes.byref(peak_ms)))
    peak = peak_tf.value

    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    width = max(max(len(s) for s in shards), 1)  # all-gather needs equal sizes
    prob = DeviceProblem(lib, at, dg, nh, False, dev, stream, max_ranges=width)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    gathered = [torch.zeros(width, dtype=torch.complex128, device=dev) for _ in shards]

    def step(arith, ev_terms=None):
        prob.launch(mine, arith, ev_terms)
        gather_shards(prob.d_part, gathered, dist)

    for _ in range(args.warmup):
        step(args.arith)
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
        step(args.arith, et)
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
    total_max, _ = max_over_ranks([total_s, terms_s], dist, dev)
    result = assemble(shards, gathered, None if dist is not None else prob.d_part)
    value = args.steps * nterms / total_max
    achieved = my_flops / (terms_s / args.steps) / 1e12
    step_sec = total_max / args.steps

    # e2e: host inputs through the public API, wall clock (incl. H2D / D2H every step)
    e2e_times = []
    h2d = (at.nbytes + dg.nbytes)
    d2h = 16 * max(len(mine), 1) + 8 * max(len(mine), 1)
    e2e_steps = max(1, min(args.steps, 5))
    for k in range(1 + e2e_steps):
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        if world == 1:
            engine.hafnian(A, backend="charpoly", arith=args.arith)
        else:
            from paper_1805_12498_b200 import distributed

            distributed.sharded_hafnian(
                nh, lambda rl: kernels.sum_range_list(at, dg, nh, N_RANGES, rl, 1, False,
                                                      arith=args.arith, device=local),
                dist, rank, world)
        dt = max_over_ranks([time.perf_counter() - t0], dist, dev)[0]
        if k >= 1:
            e2e_times.append(dt)
    e2e_value = nterms / statistics.median(e2e_times)

    # bit-exact MIRROR arithmetic on the same step (reported beside the headline)
    mirror = None
    if args.mirror_steps > 0:
        m_ms = []
        for _ in range(args.mirror_steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step("mirror")
            e1.record(stream)
            torch.cuda.synchronize()
            m_ms.append(e0.elapsed_time(e1))
        m_s = max_over_ranks([max(m_ms) / 1e3], dist, dev)[0]
        mres = assemble(shards, gathered, None if dist is not None else prob.d_part)
        mirror = {"value": nterms / m_s, "unit": UNIT, "sec_per_hafnian": m_s,
                  "steps": args.mirror_steps, "result": [mres.real, mres.imag],
                  "rel_diff_fast_vs_mirror": abs(result - mres) / abs(mres) if mres else None,
                  "note": "arith=mirror reproduces the reference's IEEE operation sequence; its "
                          "terms and partials are bit-identical to hafnium's numba kernels "
                          "(tests/test_gpu_parity.py)"}

    ref_cache = _referee() if rank == 0 else {}
    threads = len(os.sched_getaffinity(0))
    cref = None
    if rank == 0 and world == 1:
        try:
            cref = NumbaReference(threads)
        except ImportError:
            cref = None

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

    # the reference's DEFAULT backend (spectral: Hessenberg + shifted QR) on the identical
    # range [0, 2^20) of this workload: FAST spectral, bit-exact MIRROR spectral, and the
    # unmodified reference / the C port on the host cores
    spectral = None
    if rank == 0 and world == 1 and args.spectral_bits > 0:
        spectral = run_spectral(at, dg, nh, local, args, cref, threads, ref_cache)

    # per-config legs and the multi-GPU proxy (one GPU, rank 0 of a single-rank run)
    configs = proxy = None
    if rank == 0 and world == 1 and not args.no_configs:
        configs = run_configs(lib, dev, stream, peak, cref, threads, ref_cache)
    if rank == 0 and world == 1 and not args.no_proxy:
        proxy = run_proxy(lib, at, dg, nh, dev, stream, step_sec)

    # parity: (1) against the extended-precision referee (the truth) on this workload;
    # (2) north star at full size: identical contiguous range [0, 2^20), FAST and MIRROR
    # against the CPU oracle (bit-pinned to the reference)
    parity = None
    if rank == 0 and args.parity_bits > 0:
        from oracle import oracle as O
        from paper_1805_12498_b200 import accuracy

        O.build()
        hi = 1 << min(args.parity_bits, nh)
        masks = np.arange(1, hi, dtype=np.uint64)
        t_orc = O.terms(at, dg, nh, masks, backend=1, threads=threads)[0]
        t_fast, _ = kernels.terms(at, dg, nh, masks, 1, False, arith="fast", device=local)
        t_mir, _ = kernels.terms(at, dg, nh, masks, 1, False, arith="mirror", device=local)
        n_ch = 512
        r_orc = O.tree_reduce(O.sum_mask_range(at, dg, nh, 0, hi, n_ch, 1, False)[0])
        r_fast = engine.tree_reduce(kernels.sum_mask_range(at, dg, nh, 0, hi, n_ch, 1, False,
                                                           arith="fast", device=local)[0])
        r_mir = engine.tree_reduce(kernels.sum_mask_range(at, dg, nh, 0, hi, n_ch, 1, False,
                                                          arith="mirror", device=local)[0])
        abs_sum = float(np.abs(t_orc).sum())
        den = np.maximum(np.abs(t_orc), 1e-300)
        parity = {
            "tolerance": {"rel": accuracy.REL, "abs_sum": accuracy.ABS_SUM,
                          "rule": "|x - truth| <= max(1e-10 |truth|, 5e-15 sum|t|), truth = the "
                                  "long double referee (oracle/referee.c); the reference itself "
                                  "meets this and misses plain 1e-10 (paper_1805_12498_b200/"
                                  "accuracy.py); MIRROR must be bit-identical to the reference"},
            "range": f"masks [0, 2^{min(args.parity_bits, nh)}) of the n={args.n} workload, "
                     f"{n_ch} Kahan chunks + fixed tree (SURVEY.md 8(c) harness)",
            "oracle": "oracle/hafnian_oracle.c (bit-identical to hafnium.kernels._numba on the "
                      "golden fixtures), charpoly backend",
            "fast_rel_diff_vs_reference": abs(r_fast - r_orc) / abs(r_orc),
            "fast_max_term_rel_diff_vs_reference": float((np.abs(t_fast - t_orc) / den).max()),
            "mirror_bit_identical_result": bool(r_mir == r_orc),
            "mirror_bit_identical_terms": int((np.ascontiguousarray(t_mir).view(np.uint64).reshape(-1, 2)
                                               == np.ascontiguousarray(t_orc).view(np.uint64).reshape(-1, 2))
                                              .all(axis=1).sum()),
            "terms": int(masks.size),
            "cond_abs_sum_over_result": abs_sum / abs(r_orc),
        }
        key = f"range_n{args.n}s{args.seed}"
        if args.parity_bits == 20 and key in ref_cache:
            parity["range_vs_referee"] = {"fast": _score(r_fast, ref_cache, key),
                                          "mirror_eq_reference": _score(r_mir, ref_cache, key)}
        if args.n == 52 and args.seed == 3 and "full_n52s3" in ref_cache:
            R = ref_cache["full_n52s3"]
            full = {"hi": R["hi"], "lo": R["lo"], "abs_sum": R["abs_sum"]}
            parity["full_hafnian_vs_referee"] = {
                "fast": _score(result, {"f": full}, "f"),
                "mirror_eq_reference": (_score(complex(*mirror["result"]), {"f": full}, "f")
                                        if mirror else None)}
        if configs:
            parity["configs_vs_referee"] = {k: v.get("accuracy") for k, v in configs.items()}
        ok = [parity["mirror_bit_identical_result"]]
        for blk in ("range_vs_referee", "full_hafnian_vs_referee"):
            for v in (parity.get(blk) or {}).values():
                if v:
                    ok.append(v["within_bound"])
        parity["pass"] = all(ok)

    cpu = None
    if rank == 0 and world == 1:
        prate, pcount, pdt = port_rate(at, dg, nh, min(3.0, args.cpu_seconds), threads)
        port = {"value": prate, "unit": UNIT, "cores": threads, "kind": "port",
                "sample": f"{pcount} uniform random masks ({pdt:.1f} s); oracle/hafnian_oracle.c"}
        if cref is not None:
            rate, count, dt = cref.rate(at, dg, nh, 1, args.cpu_seconds, seed=7)
            cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"{count} uniform random masks of the n={args.n} problem ({dt:.1f} s) "
                             f"through the unmodified reference (baseline/_ref hafnium, numba "
                             f"kernels, charpoly backend); full hafnian extrapolated "
                             f"{nterms / rate:.0f} s",
                   "cpu": cpu_model(), "port": port}
        else:
            cpu = dict(port, cpu=cpu_model())

    traffic = None
    tpath = os.path.join(REPO, "profiles", "roofline_traffic.json")
    if os.path.exists(tpath):
        try:
            # measured DRAM bytes per term of the term kernels (profiles/roofline_traffic.json),
            # per launch-set of one step
            traffic = json.load(open(tpath)).get("bytes_per_term") * nterms
        except (ValueError, OSError, TypeError):
            traffic = None

    if rank == 0:
        line = {
            "metric": metric_name(args.n), "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * step_sec,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64 (complex128)", "data": "synthetic (seeded, SURVEY.md Appendix A)",
            "config": config(args, world),
            "sec_per_hafnian": step_sec,
            "result": [result.real, result.imag],
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak,
                         "frac_nominal": achieved / NOMINAL_FP64_TFLOPS,
                         "nominal_peak": NOMINAL_FP64_TFLOPS, "traffic": traffic,
                         "peak_source": f"DFMA probe measured in this run (hafb_fp64_peak, "
                                        f"{peak_ms.value:.2f} ms); MEASURED_PEAKS.json has no "
                                        f"FP64 entry",
                         "flop_model": "SURVEY.md 8(d) CMA model, 8 FLOP per complex MAC"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clk,
        }
        for k, v in (("mirror", mirror), ("spectral", spectral), ("exact", exact_line), ("configs", configs),
                     ("multi_gpu_proxy", proxy), ("parity", parity), ("cpu_baseline", cpu)):
            if v is not None:
                line[k] = v
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
