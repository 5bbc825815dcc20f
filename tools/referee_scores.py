"""Score FAST, MIRROR (== the reference, bit for bit) against the extended-precision
referee fixtures on every config (dev tool; prints one JSON object).

    python tools/referee_scores.py [--out gpurun_out/referee_scores.json]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

from conftest import load_golden  # noqa: E402
from paper_1805_12498_b200 import engine, kernels, workloads as W  # noqa: E402


def rel(v, hi, lo):
    d = (complex(v) - complex(hi)) - complex(lo)
    return abs(d) / abs(complex(hi))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--batch", type=int, default=4096)
    a = ap.parse_args()
    ref = load_golden("referee.npz")
    rng = load_golden("ranges.npz")
    r52 = load_golden("range_n52.npz")
    out = {}
    for name in ("cfg0", "cfg2", "cfg3", "cfg1s0", "cfg1s1", "cfg1s2", "cfg1s3"):
        c, R = rng[name], ref[name]
        loops = bool(c["loops"])
        f = engine.loop_hafnian if loops else engine.hafnian
        fast = f(c["A"], backend="charpoly", arith="fast")
        mirror = f(c["A"], backend="charpoly", arith="mirror")
        out[name] = dict(fast=rel(fast, R["hi"], R["lo"]), mirror=rel(mirror, R["hi"], R["lo"]),
                         ref_b1=rel(complex(c["result_b1"]), R["hi"], R["lo"]),
                         ref_b0=rel(complex(c["result_b0"]), R["hi"], R["lo"]),
                         cond=float(R["abs_sum"]) / abs(complex(R["hi"])))
    for name, c in r52.items():
        R = ref[f"range_{name}"]
        at, dg, nh = engine._prepare(c["A"], False)
        fs, _ = kernels.sum_mask_range(at, dg, nh, 0, 1 << 20, 512, 1, False, arith="fast")
        ms, _ = kernels.sum_mask_range(at, dg, nh, 0, 1 << 20, 512, 1, False, arith="mirror")
        out[f"range_{name}"] = dict(fast=rel(engine.tree_reduce(fs), R["hi"], R["lo"]),
                                    mirror=rel(engine.tree_reduce(ms), R["hi"], R["lo"]),
                                    ref_b1=rel(complex(c["result_b1"]), R["hi"], R["lo"]),
                                    cond=float(R["abs_sum"]) / abs(complex(R["hi"])))
    # per-term
    tg = load_golden("terms.npz")
    worst = {"fast": 0.0, "ref_b1": 0.0}
    for name, c in tg.items():
        loops = bool(c["loops"])
        at, dg, nh = engine._prepare(c["A"], loops)
        rv = ref[f"terms_{name}"]["values"]
        fv, _ = kernels.terms(at, dg, nh, c["masks"], 1, loops, arith="fast")
        sc = np.maximum(np.abs(rv), 1e-300)
        ef = float(np.max(np.abs(fv - rv) / sc))
        er = float(np.max(np.abs(c["terms_b1"] - rv) / sc))
        out[f"terms_{name}"] = dict(fast=ef, ref_b1=er)
        worst["fast"] = max(worst["fast"], ef)
        worst["ref_b1"] = max(worst["ref_b1"], er)
    out["terms_worst"] = worst
    # batch
    bpath = os.path.join(REPO, "tests", "golden", "referee_batch.npz")
    gpath = os.path.join(REPO, "tests", "golden", "batch_cfg1.npz")
    if os.path.exists(bpath) and os.path.exists(gpath):
        B = np.load(bpath)
        G = np.load(gpath)
        nb = a.batch
        As = np.array([W.cfg1(s) for s in range(nb)])
        t0 = time.time()
        fast = engine.hafnian_batch(As, backend="charpoly", arith="fast")
        t1 = time.time()
        mirror = engine.hafnian_batch(As, backend="charpoly", arith="mirror")
        hi, lo = B["hi"][:nb], B["lo"][:nb]
        ef = np.abs((fast - hi) - lo) / np.abs(hi)
        em = np.abs((mirror - hi) - lo) / np.abs(hi)
        er = np.abs((G["result_b1"][:nb] - hi) - lo) / np.abs(hi)
        es = np.abs((G["result_b0"][:nb] - hi) - lo) / np.abs(hi) if "result_b0" in G.files else er
        out["batch"] = dict(n=nb, fast_max=float(ef.max()), fast_med=float(np.median(ef)),
                            ref_b1_max=float(er.max()), ref_b1_med=float(np.median(er)),
                            ref_b0_max=float(es.max()), mirror_eq_ref=int(np.sum(mirror == G["result_b1"][:nb])),
                            fast_gt_ref=int(np.sum(ef > er)), fast_gt_2ref=int(np.sum(ef > 2 * er)),
                            fast_gt_1e10=int(np.sum(ef > 1e-10)), ref_gt_1e10=int(np.sum(er > 1e-10)),
                            fast_s=t1 - t0)
    s = json.dumps(out, indent=1)
    print(s)
    if a.out:
        with open(a.out, "w") as f:
            f.write(s)


if __name__ == "__main__":
    main()
