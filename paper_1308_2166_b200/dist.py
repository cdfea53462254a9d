"""Estimator sharding across processes (one per GPU) -- the multi-GPU plumbing of the bulk update.

Estimators are independent units (PAPER.md:105-136 contrasts the per-processor schemes; the coordinated
bulk update of PAPER.md:142-162 applies to any subset of estimators), so rank g of G owns the contiguous
global ids [floor(g r / G), floor((g+1) r / G)) and runs the whole per-batch update for them.  Because
every random draw is keyed by the GLOBAL estimator id (reading R7), the union of the shards is
bit-identical to one unsharded run.  The only exchanges are

* the batch itself, broadcast from rank 0 (NCCL over NVLink on GPUs; gloo in the CPU tests), and
* the exact partial sums S_g = sum of chi over closed estimators, all-reduced once per estimate
  (the estimate is m * S / r, reading R9).

torch.distributed is plumbing only: every step of the update runs in the engine (the CUDA library via
TriangleCounter; tests may plug in the CPU oracle to exercise this module on gloo).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(r: int, rank: int, world: int) -> tuple[int, int]:
    """(first, count) of rank's contiguous share of r estimators."""
    if not (0 <= rank < world) or r < 1:
        raise ValueError("bad shard request")
    first = rank * r // world
    return first, (rank + 1) * r // world - first


class ShardedCounter:
    """This rank's shard of r estimators behind the same push/estimate interface as TriangleCounter.

    engine_factory(r, seed, first, count) builds the per-rank engine (default: the CUDA library on the
    current device).  `buffer` is where broadcast batches land: a (w_max, 2) int32 tensor on the device
    the process group's backend serves (cuda for NCCL, cpu for gloo).
    """

    def __init__(self, r: int, seed: int, w_max: int, device=None, engine_factory=None, group=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.r, self.seed = int(r), int(seed)
        self.first, self.count = shard(self.r, self.rank, self.world)
        if engine_factory is None:
            from . import TriangleCounter
            dev = torch.cuda.current_device() if device is None else device
            engine_factory = lambda r_, s_, f_, c_: TriangleCounter(r_, s_, first=f_, count=c_, device=dev,  # noqa: E731
                                                                   w_max_hint=w_max)
        self.engine = engine_factory(self.r, self.seed, self.first, self.count)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else "cpu"
        self.buffer = torch.empty((int(w_max), 2), dtype=torch.int32, device=device)
        self.m = 0

    def push_batch(self, edges, w: int | None = None):
        """Rank 0 passes the batch (a (w, 2) uint32/int32 tensor or array); the others pass None.  Unless
        every rank passes w, the batch size is broadcast first; then the edges into `buffer`, then every
        rank updates its shard."""
        if self.world > 1:
            with self._on_engine_stream():
                if w is None:
                    n = torch.tensor([0 if edges is None else len(edges)], dtype=torch.int64, device=self.buffer.device)
                    dist.broadcast(n, src=0, group=self.group)
                    w = int(n.item())
                if w > self.buffer.shape[0]:
                    raise ValueError("batch larger than w_max")
                if self.rank == 0:
                    src = torch.as_tensor(edges) if not isinstance(edges, torch.Tensor) else edges
                    self.buffer[:w].copy_(src.view(torch.int32).reshape(w, 2))
                dist.broadcast(self.buffer[:w], src=0, group=self.group)
            batch = self.buffer[:w]
        else:
            batch = edges
            w = len(edges)
        if w == 0:
            return 0
        eng_in = batch if self.buffer.device.type != "cpu" else batch.numpy().view("uint32")
        rc = self.engine.push_batch(eng_in)
        if rc != 0:
            raise RuntimeError(f"push_batch failed on rank {self.rank}: {rc}")
        self.m += w
        return rc

    def _on_engine_stream(self):
        """The broadcast runs on the engine's own CUDA stream, so the update kernels that read the batch are
        ordered after it and the next broadcast after them (no host synchronisation)."""
        ptr = getattr(self.engine, "stream_ptr", 0) if self.buffer.device.type == "cuda" else 0
        if not ptr:
            import contextlib
            return contextlib.nullcontext()
        return torch.cuda.stream(torch.cuda.ExternalStream(ptr, device=self.buffer.device))

    def closed_sum(self) -> int:
        """S over ALL ranks (exact integer all-reduce of the per-rank partial sums)."""
        s = torch.tensor([self.engine.closed_sum()], dtype=torch.int64, device=self.buffer.device)
        if self.world > 1:
            dist.all_reduce(s, op=dist.ReduceOp.SUM, group=self.group)
        return int(s.item())

    def estimate(self) -> float:
        """m * S / r as one fixed fp64 expression (reading R9) -- identical on every rank."""
        return float(self.m) * float(self.closed_sum()) / float(self.r)
