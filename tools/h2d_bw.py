"""H2D bandwidth from pinned memory: one copy vs the same bytes split over 2 or 4 streams (copy engines)."""
import torch

n = 8 << 20
src = torch.empty(n, dtype=torch.uint8).pin_memory()
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
for k in (1, 2, 4):
    best = 1e9
    for rep in range(20):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        evs = []
        for i in range(k):
            s = streams[i]
            s.wait_event(e0)
            with torch.cuda.stream(s):
                lo, hi = i * n // k, (i + 1) * n // k
                dst[lo:hi].copy_(src[lo:hi], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s)
                evs.append(ev)
        for ev in evs:
            torch.cuda.current_stream().wait_event(ev)
        e1.record()
        e1.synchronize()
        if rep > 2:
            best = min(best, e0.elapsed_time(e1))
    print(f"{k} stream(s): {n / best / 1e6:.1f} GB/s ({best * 1e3:.0f} us for {n >> 20} MiB)")
