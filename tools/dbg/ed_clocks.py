"""k_ed_process per-item phase clocks (build with -DTC_ED_CLOCKS into libtc_clk.so)."""
import ctypes as C, sys
import numpy as np, torch
from synth import config_stream
from paper_1308_2166_b200 import TriangleCounter, _lib
w = 4096; start = 8000; n = 200
s = config_stream("C5")
dev = torch.from_numpy(s.view(np.int32)).cuda()
tc = TriangleCounter(1 << 22, 42, w_max_hint=w); tc.set_mode("event"); tc.set_async(True)
L = _lib.load()
buf = np.zeros((1 << 22, 8), np.uint32)
for k in range(start):
    tc.push_batch(dev[k * w:(k + 1) * w])
assert tc.sync() == 0
L.tc_debug_ed_clocks(buf.ctypes.data_as(C.c_void_p), 1 << 22, 1)
per = []
for k in range(start, start + n):
    tc.push_batch(dev[k * w:(k + 1) * w])
    assert tc.sync() == 0
    m = L.tc_debug_ed_clocks(buf.ctypes.data_as(C.c_void_p), 1 << 22, 1)
    per.append(buf[:m].copy())
allr = np.concatenate(per)
tot = allr[:, 4].astype(np.float64)
ph = np.diff(np.concatenate([np.zeros((len(allr), 1)), allr[:, :5].astype(np.float64)], axis=1), axis=1)
ev = allr[:, 6].astype(np.int64) - allr[:, 7].astype(np.int64)
print("items", len(allr), "mean cycles", tot.mean(), "p50", np.percentile(tot, 50), "p99", np.percentile(tot, 99), "max", tot.max())
print("mean phase cycles [load+vinfo, epochs, closure, S/ncl, rearm]", ph.mean(0).round(0))
mx = np.array([p[:, 4].max() for p in per])
print("per-batch max cycles mean", mx.mean(), "-> us at 1.965 GHz", mx.mean() / 1965)
idx = np.argsort(-tot)[:20]
for i in idx[:10]:
    print("slow item: phases", ph[i].round(0), "events", ev[i])
for e in range(0, 6):
    sel = ev == e
    if sel.any(): print("events", e, "count", sel.sum(), "mean cycles", tot[sel].mean().round(0))
