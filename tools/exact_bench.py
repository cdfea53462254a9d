"""Timing of tc_exact_triangles on a config stream (device-resident edges): device ms per call and edges/s.
Usage: python tools/exact_bench.py --config C2 [--reps 3]"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1308_2166_b200 import exact_triangles  # noqa: E402
from synth import config_stream  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch
    s = config_stream(args.config)
    dev = torch.from_numpy(s.view(np.int32)).cuda()
    res = [exact_triangles(dev, timing=True) for _ in range(args.reps + 1)][1:]
    ms = min(r[1] for r in res)
    print(json.dumps({"config": args.config, "m": len(s), "tau": res[0][0], "device_ms": ms,
                      "edges_per_s": len(s) / (ms * 1e-3)}))


if __name__ == "__main__":
    main()
