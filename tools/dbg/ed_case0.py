import numpy as np, sys
sys.path.insert(0, "tests")
from synth import er, rmat
from paper_1308_2166_b200 import TriangleCounter
from oracle.edc import EventOracleC
case = int(sys.argv[1]) if len(sys.argv) > 1 else 0
rng = np.random.default_rng(case)
s = er(300, 6000, case) if case % 2 == 0 else rmat(11, 4, case)[:6000]
s = np.ascontiguousarray(s, dtype=np.uint32)
r = [1, 37, 2000, 5000][case % 4]
tc = TriangleCounter(r, 100 + case); tc.set_mode("event")
o = EventOracleC(r, 100 + case)
k = 0; hist = []
prev = None
while k < len(s):
    w = int(rng.choice([1, 7, 64, 500, 1500, 4096])); hi = min(len(s), k + w)
    tc.push_batch(s[k:hi]); o.push_batch(s[k:hi], validate=False)
    hist.append((k, hi))
    st, ost = tc.state(), o.state(); ev = tc.event_state()
    bad = np.nonzero((st["p1"] != ost["p1"]) | (st["p2"] != ost["p2"]) | (st["c"] != ost["c"]) | (st["closed"] != ost["closed"]) | (ev["J"] != ost["J"]) | (ev["K"] != ost["K"]) | (ev["ev"] != ost["ev"]))[0]
    if len(bad):
        i = bad[0]
        print("mismatch after batch", (k, hi), "w", hi - k, "n bad", len(bad), "est", i)
        print(" gpu:", {f: st[f][i] for f in st}, {f: ev[f][i] for f in ev})
        print(" orc:", {f: ost[f][i] for f in ost})
        if prev: print(" prev gpu:", prev[0][i] if prev else None)
        print(" counters", tc.event_counters())
        print(" last batches", hist[-6:])
        break
    prev = ({f: (st[f], ev.get(f)) for f in st},)
    prev = [{**{f: st[f][j] for f in st}, **{f: ev[f][j] for f in ev}} for j in range(min(r, 4))]
    k = hi
else:
    print("all ok", tc.event_counters())
