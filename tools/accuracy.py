"""Accuracy study on the synthetic configurations, the paper's methodology:
five trials per r, mean deviation MD% = mean over trials of |estimate - tau| / tau * 100 (PAPER.md:993-1003,
Table 2 caption), r = 200K, 2M, 20M (Table 2's columns).  tau comes from tc_exact_triangles on the GPU.
Every trial streams the whole config stream through tc_push_batch in batches of the config's w, with a
different seed; the estimate is m * S / r (tc_estimate) and, for comparison, the median of means over
16 groups (tc_estimate_mom).  The paper's theoretical sufficient r, 96 / eps^2 * m Delta / tau * ln(1/delta),
is reported beside the measured MD (the paper makes the same comparison).

Usage (GPU box): python tools/accuracy.py --configs C2 C3 --out profiles/accuracy_r01.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1308_2166_b200 import TriangleCounter, exact_triangles, required_estimators  # noqa: E402
from synth import CONFIGS, config_stream  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["C2"])
    ap.add_argument("--r", nargs="+", type=int, default=[200_000, 2_000_000, 20_000_000])
    ap.add_argument("--trials", type=int, default=5)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import torch
    out = {"method": "MD% = mean_trials |est - tau| / tau * 100 (PAPER.md:993-1003, Table 2); estimate = m S / r",
           "configs": {}}
    for name in args.configs:
        cfg = CONFIGS[name]
        t0 = time.time()
        stream = config_stream(name)
        m, w = len(stream), cfg["w"]
        gen_s = time.time() - t0
        dev = torch.from_numpy(stream.view(np.int32)).cuda()
        tau, ex_ms = exact_triangles(dev, timing=True)
        tau2, ex_ms2 = exact_triangles(dev, timing=True)  # second call: warm
        assert tau2 == tau
        deg = np.bincount(stream.ravel().astype(np.int64))
        Delta = int(deg.max())
        rec = {"desc": cfg["desc"], "m": m, "w": w, "tau": tau, "Delta": Delta, "m_Delta_over_tau": m * Delta / tau,
               "exact_device_ms": round(min(ex_ms, ex_ms2), 3),
               "exact_edges_per_s": m / (min(ex_ms, ex_ms2) * 1e-3), "gen_s": round(gen_s, 1), "runs": []}
        print(f"{name}: m={m} tau={tau} Delta={Delta} exact {min(ex_ms, ex_ms2):.1f} ms", flush=True)
        for r in args.r:
            ests, moms, times = [], [], []
            for trial in range(args.trials):
                tc = TriangleCounter(r, 1000 + trial, w_max_hint=w)
                torch.cuda.synchronize()
                t1 = time.time()
                for k in range(0, m, w):
                    tc.push_batch(dev[k:k + w], check=False)
                tc.sync()
                times.append(time.time() - t1)
                ests.append(tc.estimate())
                moms.append(tc.estimate_mom(16))
                tc.close()
            ests, moms = np.array(ests), np.array(moms)
            md = float(np.mean(np.abs(ests - tau)) / tau * 100)
            md_mom = float(np.mean(np.abs(moms - tau)) / tau * 100)
            eps = max(md / 100, 1e-6)
            run = {"r": r, "trials": args.trials, "estimates": ests.tolist(), "MD_pct": round(md, 3),
                   "MD_pct_mom16": round(md_mom, 3), "median_stream_s": round(float(np.median(times)), 4),
                   "theory_r_for_eps_eq_MD_delta_0.1": required_estimators(eps, 0.1, m, Delta, tau)}
            rec["runs"].append(run)
            print(f"  r={r:>9}: MD {md:7.3f}%  MoM16 {md_mom:7.3f}%  stream {run['median_stream_s']:.3f} s", flush=True)
        out["configs"][name] = rec
        del dev
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)
    print(json.dumps({k: [(x["r"], x["MD_pct"]) for x in v["runs"]] for k, v in out["configs"].items()}))


if __name__ == "__main__":
    main()
