import numpy as np, sys
sys.path.insert(0, "tests")
from synth import rmat
from paper_1308_2166_b200 import TriangleCounter
from oracle.edc import EventOracleC
s = np.ascontiguousarray(rmat(12, 8, 3)[:30000], dtype=np.uint32)
o = EventOracleC(3000, 5); o.push_batch(s, validate=False)
print("oracle S", o.closed_sum())
def bat(rng, m, sizes):
    out, k = [], 0
    while k < m:
        w = int(rng.choice(sizes)); out.append((k, min(m, k + w))); k += w
    return out
for sizes in ([30000], [1000], [4096], [17, 999, 5000], [5000], [8192]):
    tc = TriangleCounter(3000, 5); tc.set_mode("event")
    rng = np.random.default_rng(len(sizes))
    Ss = []
    for lo, hi in bat(rng, len(s), sizes):
        tc.push_batch(s[lo:hi])
        st = tc.state()
        Ss.append((hi, tc.closed_sum(), int(st["c"][st["closed"] == 1].astype(np.int64).sum())))
    bad = [x for x in Ss if x[1] != x[2]]
    print(sizes, "final", Ss[-1], "first bad", bad[:3], tc.event_counters())
