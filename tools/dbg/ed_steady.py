"""Event mode at C5: per-kernel averages over a steady window (after the early full sweeps)."""
import sys, time, json
import numpy as np, torch
from synth import config_stream
from paper_1308_2166_b200 import TriangleCounter
w = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
start, n = int(sys.argv[2]) if len(sys.argv) > 2 else 2000, int(sys.argv[3]) if len(sys.argv) > 3 else 1000
s = config_stream("C5")
dev = torch.from_numpy(s.view(np.int32)).cuda()
tc = TriangleCounter(1 << 22, 42, w_max_hint=w); tc.set_mode("event"); tc.set_async(True)
t0 = time.time()
for k in range(start):
    tc.push_batch(dev[k * w:(k + 1) * w])
assert tc.sync() == 0
print("prefix", start, "batches", round(time.time() - t0, 2), "s", tc.event_counters())
c0 = tc.event_counters()
tc.profile(True)
for k in range(start, start + n):
    tc.push_batch(dev[k * w:(k + 1) * w])
assert tc.sync() == 0
c1 = tc.event_counters()
pk = tc.profile_kernels()
print(json.dumps({k: round(v[0] / max(v[1], 1) * 1e3, 1) for k, v in pk.items() if v[1]}))
print({k: (c1[k] - c0[k]) / n for k in c1})
