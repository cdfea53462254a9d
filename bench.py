#!/usr/bin/env python
"""Benchmark of the per-batch update of r neighborhood-sampling estimators (bulkUpdateAll,
PAPER.md:494-505) on B200.

One step = one tc_push_batch of the next w edges of the synthetic stream (all SURVEY 8(a) rows: staging,
incidence index, edge-pair hash, fused Steps 1-3 + partial sums).  BASELINE.json's metric names no config,
so the N = 1 workload is the largest single-GPU config, configs[2] = C3 (Chung-Lu gamma 2.1, 3M vertices,
117M edges, r = 2^22, w = 2^23: 14 batches per stream).  Steps run through the stream in order; when it is
exhausted a new pass starts from a reset estimator set (the reset is untimed).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl reference]

Multi-GPU (torchrun, one process per GPU): estimators are sharded by global id; rank 0 holds the stream
and broadcasts each batch over NCCL inside the timed region; the estimate all-reduces the per-rank exact
partial sums.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
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
    ap.add_argument("--steps", type=int, default=28)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--w", type=int, default=0, help="override the batch size (C5 sweep)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--tune", action="append", default=[], help="index-geometry knob key=value (tc_tune)")
    ap.add_argument("--no-graphs", action="store_true", help="plain stream launches instead of one CUDA graph per push")
    ap.add_argument("--no-profile-pass", action="store_true", help="skip the per-kernel attribution pass")
    ap.add_argument("--cpu-batches", type=int, default=0, help="batches in the cpu_baseline sample (0: auto)")
    ap.add_argument("--mode", default="bulk", choices=["bulk", "event"],
                    help="estimator update rule (tc_set_mode): the paper's bulkUpdateAll, or the event-driven mode "
                         "(SURVEY 8(f) row 4)")
    ap.add_argument("--whole-stream", action="store_true",
                    help="time every batch of one pass over the stream (steps = batches per stream)")
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


def committed_ncu(config):
    """Per-kernel DRAM traffic and L2 hit rates for this config from the committed ncu capture
    (profiles/ncu_pipeline_<config>.json: application replay with --cache-control none, so each kernel is
    measured with the L2 contents the pipeline leaves it), or {}."""
    p = os.path.join(ROOT, "profiles", f"ncu_pipeline_{config}.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


def cpu_info():
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count()


# --------------------------------------------------------------------------------------------------
# Algorithmic bytes (SURVEY 8(d) byte model): what each kernel MUST move, per launch.
#   Ke (staging): read the batch 8 B/edge, write E 8 B/edge  -> k_count; write 2 arcs x 8 B -> k_scatter
#   Ki (index)  : 8 B per arc grouped + 16 B per distinct vertex (16w + 16D)  -> k_vhash, k_vhub (+k_vbig)
#   Kp (pairs)  : read E 8 B/edge + one 16 B pair slot per edge (24w)        -> k_pairs
#   Ku (update) : 24 B per estimator (read r1, c, r2 20 B, write c 4 B) + 16 B per replaced r1 (r1, p1)
#                 + 16 B per replaced r2 (r2, p2): B_est = 24 + 16 (P_r1 + P_r2)
#   k_scan_*, k_split: 0 (implementation overhead of the grouping; it shows up as a lower fraction)
# Whole step, the minimal model: w B_edge + R B_est with B_edge = 40 + 16 D/w.
def kernel_bytes(kernel, w, st, R):
    arcs = 2 * w
    if kernel == "k_count":
        return 16 * w
    if kernel == "k_scatter":
        return 16 * w
    if kernel == "k_pairs":
        return 24 * w
    if kernel == "k_vhash":
        return 8 * (arcs - st["arcs_big"]) + 16 * (st["vertices"] - st["vertices_big"])
    if kernel == "k_vhub":
        return 8 * st["arcs_big"] + 16 * st["vertices_big"]
    if kernel == "k_small_index":  # the whole index of a small batch in one kernel: Ke 32w + Ki 16w + 16D + Kp 24w
        return 72 * w + 16 * st["vertices"]
    if kernel == "k_update":
        return 24 * R + 32 * st["fresh"] + 16 * st["r2_replaced_retained"] - 4 * st["skipped"]
    # event mode (DESIGN.md section 10 row 4): per arc the segment read, per distinct vertex a persistent-table
    # probe and the 16-byte segment record; per edge the trigger lookups (time, pair, two degree thresholds:
    # 4 x 16-byte slots) and the edge / arc records; per visited estimator its 48-byte state read and written and
    # about 4 watch nodes + map slots armed (4 x 32 B)
    if kernel == "k_ed_pre":
        return 16 * w + 48 * st["vertices"]
    if kernel == "k_ed_trigger":
        return 96 * w
    if kernel == "k_ed_front":  # k_ed_pre + k_ed_trigger in one kernel
        return 16 * w + 48 * st["vertices"] + 96 * w
    if kernel == "k_ed_process":
        return (96 + 128) * st.get("visited", 0)
    if kernel == "k_ed_post":
        return 16 * w + 32 * st["vertices"]
    return 0


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
    from paper_1308_2166_b200.dist import RankCounter
    libbuild.build()

    cfg = dict(CONFIGS[args.config])
    r = cfg["r"]
    w = args.w or cfg["w"]
    t_gen = time.perf_counter()
    stream = config_stream(args.config)
    t_gen = time.perf_counter() - t_gen
    m_total = len(stream)
    nb = (m_total + w - 1) // w
    if args.whole_stream:
        args.steps = nb
    first = rank * r // world
    count = (rank + 1) * r // world - first

    # stream resident in HBM before timing ("excluding I/O"); rank 0 owns it.  C4's ~1B
    # edges (8 GB) stay in host memory: only the e2e leg (pinned host feed) runs for it
    resident = args.config != "C4"
    dstream = torch.from_numpy(stream.view(np.int32)).to(dev) if (rank == 0 and resident) else None
    flush = torch.ones(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    flush_sink = torch.zeros((), dtype=torch.float32, device=dev)

    knobs = {k: int(v) for k, v in (kv.split("=") for kv in args.tune)}

    # one shard of the estimators per rank (tc_create_rank): the library broadcasts each batch from rank 0 with
    # NCCL over NVLink (the per-batch exchange, inside the timed step) and all-reduces the partial sums
    if world > 1:
        sc = RankCounter(r, args.seed, w, device=dev)
        tc = sc.engine
    else:
        tc = TriangleCounter(r, args.seed, device=dev.index, w_max_hint=w)
    assert (tc.first, tc.count) == (first, count)
    if args.mode == "event":
        tc.set_mode("event")
    tc.set_async(True)
    if knobs:
        tc.tune(**knobs)
    ext = torch.cuda.ExternalStream(tc.stream_ptr, device=dev)

    def push(k):
        lo, hi = (k % nb) * w, min(m_total, (k % nb) * w + w)
        if rank == 0:
            tc.push_batch(dstream[lo:hi])
        else:
            tc.push_batch(None, w=hi - lo)
        return hi - lo

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    out = {"metric": METRIC, "unit": "edges/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
           "dtype": "u32",
           "data": "synthetic (seeded native generator, synth/gen.c; the paper's SNAP datasets are not available)"}
    peak, peak_src = measured_peaks()

    if resident:
        # ---- warm-up (untimed) ----
        for k in range(args.warmup):
            if k and k % nb == 0:
                assert tc.sync() == 0
                tc.reset()
            push(k)
        assert tc.sync() == 0

        # ---- timed: K steps = K consecutive batches of the stream; CUDA events on the library's stream
        # around each step; L2 flushed (read of a 256 MiB buffer) before every step, outside the events ----
        def timed_pass(nsteps, profile, graphs):
            tc.set_graphs(graphs)
            tc.reset()
            tc.profile(profile)
            evs, launches, edges = [], 0, 0
            kern = {}
            stats = {}

            def harvest():
                if profile:
                    for name, (kms, n) in tc.profile_kernels().items():
                        acc = kern.setdefault(name, [0.0, 0])
                        acc[0] += kms
                        acc[1] += n
                for kk, v in tc.stats().items():
                    stats[kk] = stats.get(kk, 0) + v
                if args.mode == "event":
                    ec = tc.event_counters()
                    for kk in ("visited", "events", "sweeps"):
                        stats[kk] = stats.get(kk, 0) + ec[kk]

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
            return ms_, launches, edges, kern, stats, clocks, wall

        # headline: every push as one CUDA graph (--no-graphs: plain stream launches), no profiling events
        ms, launches, edges_done, _, _, clocks, t_wall = timed_pass(args.steps, False, not args.no_graphs)
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        if world > 1:
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        secs = ms / 1e3
        value = edges_done / secs
        out.update({"value": value, "ms_per_step": ms / args.steps, "gpu_launches": launches,
                    "estimator_updates_per_s": edges_done * r / secs,
                    "batch_estimator_updates_per_s": args.steps * r / secs,
                    "wall_s_timed_region": t_wall, "clocks": clocks.summary()})

        # ---- attribution: one more pass over the whole stream with CUDA events around every kernel (plain
        # launches), the per-kernel algorithmic bytes of the byte model and the event counts it needs ----
        if not args.no_profile_pass:
            _, _, prof_edges, kern, stats, _, _ = timed_pass(nb, True, False)
            nsteps = nb
            R_total = count * nsteps
            rows = {}
            for name, (kms, n) in kern.items():
                if n == 0:
                    continue
                B = kernel_bytes(name, prof_edges, stats, R_total)
                rows[name] = {"ms_per_launch": kms / n, "launches": n, "share_of_kernel_time": None,
                              "algorithmic_bytes_per_launch": B / n,
                              "achieved_GBps": (B / (kms / 1e3) / 1e9) if B and kms > 0 else None}
            ktot = sum(kern[k][0] for k in rows)
            for name in rows:
                rows[name]["share_of_kernel_time"] = kern[name][0] / ktot
                if rows[name]["achieved_GBps"]:
                    rows[name]["frac"] = rows[name]["achieved_GBps"] / peak
            dom = max(rows, key=lambda k: kern[k][0])
            per_rank = None
            if world > 1:  # per-kernel times of every rank: the replicated index build is the Amdahl term
                per_rank = [None] * world
                torch.distributed.all_gather_object(per_rank, {k: v["ms_per_launch"] for k, v in rows.items()})
            ncu = committed_ncu(args.config)
            traffic = (ncu.get("kernels", {}).get(dom) or {}).get("dram_bytes_per_launch")
            for name, row in rows.items():  # the pipeline's own DRAM bytes per launch (ncu), as a rate
                kn = ncu.get("kernels", {}).get(name) or {}
                t_, d_ = kn.get("dram_bytes_per_launch"), kn.get("duration_us")
                if t_ and d_:  # bytes and time from the same capture (ncu serialises the kernels)
                    row["dram_bytes_per_launch_ncu"] = t_
                    row["dram_GBps"] = t_ / (d_ / 1e6) / 1e9
                    row["dram_frac"] = row["dram_GBps"] / peak
            D_avg = stats["vertices"] / nsteps
            B_step = (40 * prof_edges + 16 * stats["vertices"]) / nsteps + \
                kernel_bytes("k_update", prof_edges, stats, R_total) / nsteps
            step_ms = ms / args.steps
            out["roofline"] = {
                "bound": "hbm", "kernel": dom,
                "achieved": rows[dom]["achieved_GBps"], "peak": peak, "unit": "GB/s",
                "frac": rows[dom].get("frac"), "traffic": traffic, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": rows[dom]["algorithmic_bytes_per_launch"],
                "launch_ms": rows[dom]["ms_per_launch"],
                "dram_frac": rows[dom].get("dram_frac"),
                "dram_frac_note": "traffic / duration, both from the ncu pipeline capture (DRAM bytes the kernel "
                                  "actually moves, application replay without cache control), over peak: how close "
                                  "the kernel is to HBM on the accesses it makes (a random 8-32 B probe that misses "
                                  "L2 moves a whole 128-byte line from DRAM on this part, whatever the load flavour: "
                                  "profiles/randbench_r02.txt)",
                "byte_model": "SURVEY 8(d): Ke 16w (k_count) + 16w (k_scatter); Ki 8 B/arc + 16 B/vertex; "
                              "Kp 24w; Ku 24 B/estimator + 16 B per replaced r1 + 16 B per replaced r2",
                "kernels": rows,
                "whole_step": {"algorithmic_bytes": B_step, "ms": step_ms,
                               "achieved_GBps": B_step / (step_ms / 1e3) / 1e9,
                               "frac": B_step / (step_ms / 1e3) / 1e9 / peak,
                               "model": "w (40 + 16 D/w) + R (24 + 16 (P_r1 + P_r2)) bytes (SURVEY 8(d) minimal)"},
                "events_per_batch": {"D": D_avg, "fresh_r1": stats["fresh"] / nsteps,
                                     "r2_replaced_retained": stats["r2_replaced_retained"] / nsteps,
                                     **({"visited": stats.get("visited", 0) / nsteps,
                                         "events": stats.get("events", 0) / nsteps,
                                         "full_sweeps": stats.get("sweeps", 0)} if args.mode == "event" else {})},
                "from": "CUDA events around every kernel, a second pass over the stream (plain launches); shares "
                        "agree with the committed ncu launch list profiles/launches_r02_<config>.csv",
                "per_rank_kernel_ms": per_rank,
                "l2_hit_rate_probes": (ncu.get("kernels", {}).get("k_update") or {}).get("lts_hit_rate_pct"),
                "ncu_source": ncu.get("source")}

    out["config"] = {"workload": f"{args.config}: {cfg['desc']}", "r": r, "w": w, "stream_edges": m_total,
                     "mode": args.mode, "steps_from": "stream start (one whole pass)" if args.whole_stream else
                     "stream start, consecutive batches",
                     "batches_per_stream": nb, "estimators_per_gpu": count,
                     "parallelism": f"estimator-shard x{world}",
                     "l2": "flushed before every step (256 MiB read, outside the step events)",
                     "launch": "one CUDA graph per push" if not args.no_graphs else "plain stream launches",
                     "timing": "CUDA events on the library stream around each tc_push_batch, summed; max over ranks",
                     "generation_s": round(t_gen, 2)}

    # ---- e2e: the public API with HOST (pinned) buffers, H2D + result D2H inside every step ----
    # Asynchronous errors: each push uploads its batch on the library's copy stream (overlapping the previous
    # batch's kernels) and tc_closed_sum_async copies the batch's S (the step's result) back to pinned host
    # memory; the per-step L2 flush stays inside the timed region.  CUDA events on the library stream per pass
    # over the stream; the reset between passes is untimed.
    if not args.no_e2e and world == 1:
        e_steps = args.steps if resident else min(args.steps, nb)
        host_rows = min(m_total, e_steps * w) if not resident else m_total
        host = torch.from_numpy(stream[:host_rows].view(np.int32)).pin_memory()
        if not resident:
            tc.set_graphs(not args.no_graphs)
        tc2 = tc if not resident else TriangleCounter(r, args.seed, device=dev.index, w_max_hint=w)
        if resident and args.mode == "event":
            tc2.set_mode("event")
        tc2.set_async(True)
        tc2.set_graphs(not args.no_graphs)
        ext2 = torch.cuda.ExternalStream(tc2.stream_ptr, device=dev)
        Sbuf = torch.zeros(e_steps, dtype=torch.int64).pin_memory()
        for k in range(min(args.warmup, nb)):
            tc2.push_batch(host[k * w:(k + 1) * w])
        assert tc2.sync() == 0
        tc2.reset()
        e_ms, e_edges, h2d, k, est, est_ok = 0.0, 0, 0, 0, 0.0, True
        with ClockSampler(dev.index) as clocks2:
            while k < e_steps:
                n_pass = min(nb, e_steps - k)
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
                      "h2d_bytes_per_step": h2d // e_steps, "d2h_bytes_per_step": 8, "steps": e_steps,
                      "note": "tc_push_batch(pinned host edges, asynchronous errors: H2D on the copy stream overlaps "
                              "the previous batch) + tc_closed_sum_async (8-byte S per step) + the per-step L2 flush; "
                              "CUDA events on the library stream per pass over the stream"}
        out["e2e_last_estimate"] = est
        out["e2e_results_match_tc_estimate"] = est_ok
        if not resident:  # C4: the pinned-host feed IS the workload
            out.update({"value": out["e2e"]["value"], "ms_per_step": e_ms / e_steps, "steps": e_steps,
                        "estimator_updates_per_s": e_edges * r / (e_ms / 1e3),
                        "clocks": clocks2.summary()})

    # ---- CPU baseline: the oracle as it stands, on this host's cores (rank 0, N = 1 only) ----
    if not args.no_cpu_baseline and world == 1:
        nbat = args.cpu_batches or max(1, min(8, (1 << 24) // max(w, r)))
        out["cpu_baseline"] = (cpu_baseline_event(stream, r, w, args.seed) if args.mode == "event" else
                               cpu_baseline(stream, r, w, args.seed, nbatches=min(nbat, nb)))

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
    model, ncpu = cpu_info()
    return {"value": edges / dt, "unit": "edges/s", "cores": threads(), "kind": "oracle",
            "cpu_model": model, "host_cpus": ncpu, "omp_num_threads_env": os.environ.get("OMP_NUM_THREADS"),
            "sample": f"first {nbatches} batch(es) ({edges} edges) of the same stream at full r={r}, w={w}; "
                      f"oracle/indexed.c (qsort + binary-search multisearch, OpenMP over estimators), {dt:.1f} s"}


def cpu_baseline_event(stream, r, w, seed):
    """The event mode's oracle (oracle/ed.c: every estimator walked event by event, OpenMP) on a stream prefix
    of about 2^21 edges at full r (its cost is per estimator event, so the sample is a prefix, not a batch)."""
    from oracle.edc import EventOracleC, threads
    m = min(len(stream), max(w, 1 << 21))
    o = EventOracleC(r, seed)
    t0 = time.perf_counter()
    o.push_batch(stream[:m], validate=False)
    o.closed_sum()
    dt = time.perf_counter() - t0
    model, ncpu = cpu_info()
    return {"value": m / dt, "unit": "edges/s", "cores": threads(), "kind": "oracle", "cpu_model": model,
            "host_cpus": ncpu, "sample": f"the first {m} edges of the same stream at full r={r} through oracle/ed.c "
                                         f"(event mode), {dt:.1f} s"}


def run_reference(args):
    """--impl reference: the oracle (this tier's reference arm) timed on the host cores, on the same config.
    A step is one whole batch at full r; the run is bounded to at most 3 timed steps and 1 warm-up step so
    that it ends within a few minutes at C3/C4 (a C3 batch takes the oracle ~5-10 s)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle.indexed import IndexedOracle, threads
    cfg = dict(CONFIGS[args.config])
    r = cfg["r"]
    w = args.w or cfg["w"]
    stream = config_stream(args.config)
    nb = (len(stream) + w - 1) // w
    steps = max(1, min(args.steps, 3 if w * 1.0 * r >= 2 ** 40 else args.steps))
    warm = min(args.warmup, 1)
    o = IndexedOracle(r, args.seed)
    for k in range(warm):
        o.push_batch(stream[(k % nb) * w:(k % nb) * w + w])
    o = IndexedOracle(r, args.seed)
    t0 = time.perf_counter()
    edges = 0
    for k in range(steps):
        if k and k % nb == 0:
            o = IndexedOracle(r, args.seed)
        W = stream[(k % nb) * w:(k % nb) * w + w]
        assert o.push_batch(W) == 0
        edges += len(W)
    dt = time.perf_counter() - t0
    v = edges / dt
    model, ncpu = cpu_info()
    cb = {"value": v, "unit": "edges/s", "cores": threads(), "kind": "oracle", "cpu_model": model,
          "host_cpus": ncpu, "sample": f"{steps} whole batch(es) (w={w}) of {args.config} at full r={r}"}
    print(json.dumps({"impl": "reference", "metric": METRIC, "value": v, "unit": "edges/s", "n_gpus": world,
                      "steps": steps, "steps_requested": args.steps, "warmup": warm,
                      "ms_per_step": dt * 1e3 / steps, "higher_is_better": True, "scaling": "weak",
                      "vs_baseline": None, "dtype": "u32", "data": "synthetic",
                      "config": {"workload": f"{args.config}: {cfg['desc']}", "r": r, "w": w},
                      "cpu_baseline": cb,
                      "e2e": {"value": v, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
          flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_b200(a)
