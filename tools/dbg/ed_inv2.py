import numpy as np, sys
from synth import rmat
from paper_1308_2166_b200 import TriangleCounter
s = np.ascontiguousarray(rmat(12, 8, 3)[:30000], dtype=np.uint32)
for w, knobs in ((1000, dict(small_index=1)), (1000, dict(small_index=1, vbucket_cap=64)), (5000, {}), (2000, dict(small_index=1, vbucket_arcs=64))):
    tc = TriangleCounter(3000, 5); tc.set_mode("event"); tc.tune(**knobs)
    out = []
    for k in range(0, len(s), w):
        tc.push_batch(s[k:k + w])
        st = tc.state()
        out.append((k + w, tc.closed_sum(), int(st["c"][st["closed"] == 1].astype(np.int64).sum())))
    bad = [x for x in out if x[1] != x[2]]
    print(w, knobs, "first bad", bad[:2], tc.event_counters())
