#!/usr/bin/env python
"""Benchmark of the per-batch update of r neighborhood-sampling estimators (bulkUpdateAll,
PAPER.md:494-505) on B200.

One step = one tc_push_batch of the next w edges of the synthetic stream (all §8(a) rows: staging,
incidence index, edge-pair hash, fused Steps 1-3 + partial sums).  Default workload = BASELINE.json
configs[1] (C2: R-MAT scale 20, ~15.7M edges, r = w = 2^20): the full stream is 15 batches, so the
default --steps 15 times one whole stream through a fresh estimator set.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl reference]

Multi-GPU (torchrun, one process per GPU): estimators are sharded by global id; rank 0 holds the
stream and broadcasts each batch over NCCL inside the timed region; the estimate all-reduces the
per-rank exact partial sums.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import CONFIGS, config_stream  # noqa: E402

METRIC = "edges/s and estimator-updates/s per batch; fraction of HBM roofline"
L2_FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=150)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C5"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--w", type=int, default=0, help="override the batch size (C5 sweep)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--tune", action="append", default=[], help="index-geometry knob key=value (tc_tune)")
    ap.add_argument("--no-graphs", action="store_true", help="plain stream launches instead of one CUDA graph per push")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# --------------------------------------------------------------------------------------------------
class ClockSampler:
    """SM clock and throttle reasons sampled every 5 ms DURING the timed region (NVML, the library
    nvidia-smi reads; falls back to `nvidia-smi -lms 200`)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.max_mhz = None
        self._stop = threading.Event()
        self.proc = None
        self.t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            reasons_fn = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons

            def loop():
                while not self._stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = reasons_fn(h)
                        self.rows.append((float(sm), int(rs)))
                    except Exception:
                        pass
                    time.sleep(0.005)

            self.t = threading.Thread(target=loop, daemon=True)
            self.t.start()
        except Exception:
            try:
                q = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"
                self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                              "--format=csv,noheader,nounits", "-lms", "200"],
                                             stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)

                def rd():
                    for line in self.proc.stdout:
                        f = [x.strip() for x in line.split(",")]
                        try:
                            self.max_mhz = float(f[1])
                            self.rows.append((float(f[0]), int(f[2], 16)))
                        except (ValueError, IndexError):
                            pass

                self.t = threading.Thread(target=rd, daemon=True)
                self.t.start()
            except OSError:
                pass
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return None
        sm = [r[0] for r in self.rows]
        reasons = sorted({name for _, rs in self.rows for name, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.rows), "source": "nvml" if self.proc is None else "nvidia-smi"}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def committed_traffic(config):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel, from the committed
    `ncu --set full` capture (profiles/traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f).get(config)
        if d:
            return d.get("traffic_bytes_per_launch")
    return None


def committed_limiters(kernel="k_update"):
    """What bounds the dominant kernel besides HBM, from the committed `ncu --set full` summary
    (profiles/ncu_full_r01.json): L2 throughput, issue activity, occupancy and the top stall reason."""
    p = os.path.join(ROOT, "profiles", "ncu_full_r01.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        rows = [x for x in json.load(f) if x.get("kernel", "").split("<")[0] == kernel]
    if not rows:
        return None
    x = rows[-1]

    def num(k):
        try:
            return float(str(x.get(k, "")).split()[0])
        except (ValueError, IndexError):
            return None
    return {"kernel": kernel, "lts_throughput_pct": num("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
            "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "warp_instructions_per_launch": num("smsp__inst_executed.sum"),
            "top_stall": (x.get("top_stalls") or [[None]])[0][0],
            "source": "profiles/ncu_full_r01.json (cold-L2 replay)"}


def limiters_with_issue(lim, launch_ms):
    """Add the issue-rate view: the committed capture's warp instructions per launch over this run's launch
    time, against 4 warp instructions per SM per cycle at the SM clock the recipe gives for B200
    (148 SMs x 4 x 1.965 GHz)."""
    if not lim or not lim.get("warp_instructions_per_launch") or not launch_ms:
        return lim
    peak = 148 * 4 * 1.965e9
    ach = lim["warp_instructions_per_launch"] / (launch_ms * 1e-3)
    lim = dict(lim)
    lim["issue"] = {"achieved_warp_inst_per_s": ach, "peak_warp_inst_per_s": peak, "frac": ach / peak}
    return lim


# --------------------------------------------------------------------------------------------------
def algorithmic_bytes(phase, w, R, D, fresh, r2old, skipped=0):
    """Algorithmic bytes per launch: what each phase must move at minimum.

    update    : 24 B per retained estimator (read r1 8 + cf 4 + r2 8, write cf 4), 28 B per fresh one
                (write cf 4, r1 8, p1 4, r2 8, p2 4), +12 B per retained estimator whose f2 is replaced
                (r2, p2); 20 B (no write) per estimator the small-batch pass skips as untouched; the index
                probes are not counted (the byte model of SURVEY §8d).
    partition : read the batch once 8 B/edge; write E 8, the two bucketed arcs 16, the bucketed edge 16 B/edge.
    pairs     : read the bucketed edge 16 B, write its 2 table slots 16 B.
    vertices  : read the two bucketed arcs 16 B, write segS 8 + einfo 16 B per edge; 32 B (2 slots) per vertex.
    """
    if phase == "update":
        return 24 * (R - fresh) + 28 * fresh + 12 * r2old - 4 * skipped
    if phase == "partition":
        return 48 * w
    if phase == "pairs":
        return 32 * w
    if phase == "vertices":
        return 40 * w + 32 * D
    raise KeyError(phase)


def run_b200(args):
    import torch
    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    from paper_1308_2166_b200 import TriangleCounter, build as libbuild
    from paper_1308_2166_b200.dist import ShardedCounter
    libbuild.build()

    cfg = dict(CONFIGS[args.config])
    r = cfg["r"]
    w = args.w or cfg["w"]
    stream = config_stream(args.config)
    m_total = len(stream)
    nb = (m_total + w - 1) // w
    first = rank * r // world
    count = (rank + 1) * r // world - first

    # stream resident in HBM before timing ("excluding I/O"); rank 0 owns it
    dstream = torch.from_numpy(stream.view(np.int32)).to(dev) if rank == 0 else None
    flush = torch.ones(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    flush_sink = torch.zeros((), dtype=torch.float32, device=dev)

    knobs = {k: int(v) for k, v in (kv.split("=") for kv in args.tune)}

    def engine(r_, seed_, first_, count_):
        tc_ = TriangleCounter(r_, seed_, first=first_, count=count_, device=dev.index, w_max_hint=w)
        tc_.set_async(True)
        if knobs:
            tc_.tune(**knobs)
        return tc_

    # one shard of the estimators per rank; rank 0 broadcasts each batch on the library's stream (NCCL over
    # NVLink: the per-batch exchange, inside the timed step)
    sc = ShardedCounter(r, args.seed, w, device=dev, engine_factory=engine)
    assert (sc.first, sc.count) == (first, count)
    tc = sc.engine

    def push(k):
        lo, hi = (k % nb) * w, min(m_total, (k % nb) * w + w)
        if world == 1:
            tc.push_batch(dstream[lo:hi])
        else:
            sc.push_batch(dstream[lo:hi] if rank == 0 else None, w=hi - lo)
        return hi - lo

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    # ---- warm-up (untimed) ----
    for k in range(args.warmup):
        if k and k % nb == 0:
            assert tc.sync() == 0
            tc.reset()
        push(k)
    assert tc.sync() == 0

    # ---- timed: K steps = K consecutive batches of the stream (a new pass over the stream starts from a
    # reset estimator set, untimed); CUDA events on the library's stream around each step; L2 flushed
    # (read of a 256 MiB buffer) before every step, outside the events ----
    ext = torch.cuda.ExternalStream(tc.stream_ptr, device=dev)

    def timed_pass(nsteps, profile, graphs):
        tc.set_graphs(graphs)
        tc.reset()
        tc.profile(profile)
        evs, launches, edges = [], 0, 0
        prof = {}
        stats = {"fresh": 0, "r2_replaced_retained": 0, "vertices": 0, "skipped": 0}

        def harvest():
            if profile:
                for p, (pms, n) in tc.profile_read().items():
                    acc = prof.setdefault(p, [0.0, 0])
                    acc[0] += pms
                    acc[1] += n
            for kk, v in tc.stats().items():
                if kk in stats:
                    stats[kk] += v

        barrier()
        torch.cuda.synchronize()
        with ClockSampler(dev.index) as clocks:
            t0 = time.perf_counter()
            for k in range(nsteps):
                if k and k % nb == 0:  # stream exhausted: a fresh estimator set (untimed)
                    assert tc.sync() == 0
                    harvest()
                    tc.reset()
                    tc.profile(profile)
                with torch.cuda.stream(ext):
                    flush_sink.add_(flush.sum())  # read 256 MiB (> L2): every step starts with a cold cache
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(ext)
                n = push(k)
                with torch.cuda.stream(ext):
                    e1.record(ext)
                evs.append((e0, e1))
                launches += tc.last_launches()
                edges += n
            assert tc.sync() == 0
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
        barrier()
        harvest()
        ms_ = sum(x.elapsed_time(y) for x, y in evs)
        return ms_, launches, edges, prof, stats, clocks, wall

    # headline: every push as one CUDA graph (--no-graphs: plain stream launches), no profiling events
    ms, launches, edges_done, _, _, clocks, t_wall = timed_pass(args.steps, False, not args.no_graphs)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms = float(t.item())
    secs = ms / 1e3
    # per-phase times (and the dominant kernel's launch time): one more pass over the stream with CUDA events
    # bracketing each phase (plain launches: the events are stream operations between the kernels)
    _, _, prof_edges, prof, stats, _, _ = timed_pass(nb, True, False)

    # dominant kernel = k_update (the largest single kernel in the committed ncu launch list,
    # profiles/launches_r01_summary.txt); its events bracket exactly that one launch per step
    peak, peak_src = measured_peaks()
    nsteps = nb
    alg = {
        "update": algorithmic_bytes("update", 0, count * nsteps, 0, stats["fresh"], stats["r2_replaced_retained"],
                                    stats["skipped"]),
        "partition": algorithmic_bytes("partition", prof_edges, 0, 0, 0, 0),
        "pairs": algorithmic_bytes("pairs", prof_edges, 0, 0, 0, 0),
        "vertices": algorithmic_bytes("vertices", prof_edges, 0, stats["vertices"], 0, 0),
    }
    ach = {p: alg[p] / (prof[p][0] / 1e3) / 1e9 for p in alg if prof.get(p) and prof[p][0] > 0}
    roofline = {"bound": "hbm", "kernel": "k_update (fused Steps 1-3 + partial sums)",
                "achieved": ach.get("update"), "peak": peak, "unit": "GB/s",
                "frac": ach["update"] / peak if ach.get("update") else None,
                "traffic": committed_traffic(args.config), "peak_source": peak_src,
                "algorithmic_bytes_per_launch": alg["update"] / max(1, nsteps),
                "launch_ms": prof["update"][0] / max(1, nsteps),
                "small_batch_skipped_frac": stats["skipped"] / max(1, count * nsteps),
                "limiters": limiters_with_issue(committed_limiters("k_update"), prof["update"][0] / max(1, nsteps)),
                "phases": {p: {"ms_per_step": prof[p][0] / max(1, nsteps), "launches_per_step": prof[p][1] / max(1, nsteps),
                               "algorithmic_GBps": ach.get(p), "frac": (ach[p] / peak) if ach.get(p) else None}
                           for p in prof}}

    value = edges_done / secs
    out = {
        "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded R-MAT/ER/Chung-Lu stand-ins; the paper's SNAP datasets are not available)",
        "config": {"workload": f"{args.config}: {cfg['desc']}", "r": r, "w": w, "stream_edges": m_total,
                   "batches_per_stream": nb, "estimators_per_gpu": count, "parallelism": f"estimator-shard x{world}",
                   "l2": "flushed before every step (256 MiB read, outside the step events)",
                   "launch": "one CUDA graph per push" if not args.no_graphs else "plain stream launches",
                   "phases_from": "a second pass over the stream with per-phase CUDA events (plain launches)",
                   "timing": "CUDA events on the library stream around each tc_push_batch, summed; max over ranks"},
        "estimator_updates_per_s": edges_done * r / secs,
        "batch_estimator_updates_per_s": args.steps * r / secs,
        "gpu_launches": launches,
        "roofline": roofline,
        "wall_s_timed_region": t_wall,
    }
    out["clocks"] = clocks.summary()

    # ---- e2e: the public API with HOST (pinned) buffers, H2D + result D2H inside every step ----
    # Asynchronous errors: each push uploads its batch on the library's copy stream (overlapping the previous
    # batch's kernels) and tc_closed_sum_async copies the batch's S (the step's result) back to pinned host
    # memory; the per-step L2 flush stays inside the timed region here.  Timed per pass over the stream with
    # CUDA events on the library stream; the reset between passes is untimed.
    if not args.no_e2e and world == 1:
        host = torch.from_numpy(stream.view(np.int32)).pin_memory()
        tc2 = TriangleCounter(r, args.seed, device=dev.index, w_max_hint=w)
        tc2.set_async(True)
        tc2.set_graphs(not args.no_graphs)
        ext2 = torch.cuda.ExternalStream(tc2.stream_ptr, device=dev)
        Sbuf = torch.zeros(args.steps, dtype=torch.int64).pin_memory()
        for k in range(min(args.warmup, nb)):
            tc2.push_batch(host[k * w:(k + 1) * w])
        assert tc2.sync() == 0
        tc2.reset()
        e_ms, e_edges, h2d, k, est, est_ok = 0.0, 0, 0, 0, 0.0, True
        while k < args.steps:
            n_pass = min(nb, args.steps - k)
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(ext2)
            m_run = []
            for j in range(n_pass):
                lo, hi = j * w, min(m_total, j * w + w)
                with torch.cuda.stream(ext2):
                    flush_sink.add_(flush.sum())
                tc2.push_batch(host[lo:hi])
                tc2.closed_sum_async(Sbuf, k + j)
                m_run.append(hi)
                h2d += 8 * (hi - lo)
                e_edges += hi - lo
            a1.record(ext2)
            assert tc2.sync() == 0
            e_ms += a0.elapsed_time(a1)
            est = float(m_run[-1]) * float(Sbuf[k + n_pass - 1].item()) / float(r)  # the last step's result
            est_ok = est_ok and est == tc2.estimate()
            tc2.reset()
            k += n_pass
        out["e2e"] = {"value": e_edges / (e_ms / 1e3), "unit": "edges/s",
                      "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": 8,
                      "note": "tc_push_batch(pinned host edges, asynchronous errors: H2D on the copy stream overlaps the "
                              "previous batch) + tc_closed_sum_async (8-byte S per step) + the per-step L2 flush; CUDA "
                              "events on the library stream per pass over the stream"}
        out["e2e_last_estimate"] = est
        out["e2e_results_match_tc_estimate"] = est_ok

    # ---- CPU baseline: the oracle as it stands, on this host's cores (rank 0, N = 1 only) ----
    if not args.no_cpu_baseline and world == 1:
        out["cpu_baseline"] = cpu_baseline(stream, r, w, args.seed, nbatches=min(8, nb))

    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def cpu_baseline(stream, r, w, seed, nbatches):
    from oracle.indexed import IndexedOracle, threads
    o = IndexedOracle(r, seed)
    t0 = time.perf_counter()
    edges = 0
    for k in range(nbatches):
        W = stream[k * w:(k + 1) * w]
        assert o.push_batch(W) == 0
        edges += len(W)
    dt = time.perf_counter() - t0
    return {"value": edges / dt, "unit": "edges/s", "cores": threads(), "kind": "oracle",
            "sample": f"first {nbatches} batches ({edges} edges) of the same stream at full r={r}, w={w}; "
                      f"oracle/indexed.c (qsort + binary-search multisearch, OpenMP over estimators), {dt:.1f} s"}


def run_reference(args):
    """--impl reference: the oracle (this tier's reference arm) timed on the host cores."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle.indexed import IndexedOracle, threads
    cfg = dict(CONFIGS[args.config])
    r = cfg["r"]
    w = args.w or cfg["w"]
    stream = config_stream(args.config)
    nb = (len(stream) + w - 1) // w
    o = IndexedOracle(r, args.seed)
    for k in range(args.warmup):
        if k and k % nb == 0:
            o = IndexedOracle(r, args.seed)
        o.push_batch(stream[(k % nb) * w:(k % nb) * w + w])
    o = IndexedOracle(r, args.seed)
    t0 = time.perf_counter()
    edges = 0
    for k in range(args.steps):
        if k and k % nb == 0:
            o = IndexedOracle(r, args.seed)
        W = stream[(k % nb) * w:(k % nb) * w + w]
        assert o.push_batch(W) == 0
        edges += len(W)
    dt = time.perf_counter() - t0
    v = edges / dt
    cb = {"value": v, "unit": "edges/s", "cores": threads(), "kind": "oracle",
          "sample": f"{args.steps} whole batches (w={w}) of {args.config} at full r={r}"}
    print(json.dumps({"impl": "reference", "metric": METRIC, "value": v, "unit": "edges/s", "n_gpus": world,
                      "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
                      "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
                      "data": "synthetic", "config": {"workload": f"{args.config}: {cfg['desc']}", "r": r, "w": w},
                      "cpu_baseline": cb,
                      "e2e": {"value": v, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
          flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_b200(a)
