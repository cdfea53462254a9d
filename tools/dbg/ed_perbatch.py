"""Event mode at C5: per-batch kernel times (sync after each batch) in a window, split by full-sweep batches."""
import sys, json
import numpy as np, torch
from synth import config_stream
from paper_1308_2166_b200 import TriangleCounter
w = int(sys.argv[1]); start = int(sys.argv[2]); n = int(sys.argv[3])
s = config_stream("C5")
dev = torch.from_numpy(s.view(np.int32)).cuda()
tc = TriangleCounter(1 << 22, 42, w_max_hint=w); tc.set_mode("event"); tc.set_async(True)
for k in range(start):
    tc.push_batch(dev[k * w:(k + 1) * w])
assert tc.sync() == 0
tc.profile(True)
prev = {}; prevc = tc.event_counters()
rows = []
for k in range(start, start + n):
    tc.push_batch(dev[k * w:(k + 1) * w])
    pk = tc.profile_kernels()
    c = tc.event_counters()
    row = {kk: round((v[0] - prev.get(kk, (0, 0))[0]) * 1e3, 1) for kk, v in pk.items() if v[1]}
    row["sweep"] = c["sweeps"] - prevc["sweeps"]; row["visited"] = c["visited"] - prevc["visited"]
    prev, prevc = pk, c
    rows.append(row)
sw = [r for r in rows if r["sweep"]]; ns = [r for r in rows if not r["sweep"]]
keys = [k for k in rows[0] if k.startswith("k_")]
print("non-sweep", len(ns), {k: round(np.mean([r.get(k, 0) for r in ns]), 1) for k in keys + ["visited"]})
print("non-sweep p90", {k: round(np.percentile([r.get(k, 0) for r in ns], 90), 1) for k in keys + ["visited"]})
print("sweeps", len(sw), [{k: r.get(k) for k in keys} for r in sw[:3]])
