"""Estimator sharding across processes (one per GPU) -- the multi-GPU plumbing of the bulk update.

Estimators are independent units (PAPER.md:105-136 contrasts the per-processor schemes; the coordinated
bulk update of PAPER.md:142-162 applies to any subset of estimators), so rank g of G owns the contiguous
global ids [floor(g r / G), floor((g+1) r / G)) and runs the whole per-batch update for them.  Because
every random draw is keyed by the GLOBAL estimator id (reading R7), the union of the shards is
bit-identical to one unsharded run.  The only exchanges are

* the batch itself, broadcast from rank 0 (NCCL over NVLink on GPUs; gloo in the CPU tests) -- on its own
  stream into one of two batch buffers, so batch b+1's broadcast overlaps batch b's kernels -- or, for
  host-fed batches, a 1/G slice uploaded by every rank and all-gathered, and
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

    def __init__(self, r: int, seed: int, w_max: int, device=None, engine_factory=None, group=None,
                 force_exchange: bool = False):
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
        self.device = torch.device(device)
        self.w_max = int(w_max)
        # two batch buffers: on CUDA the broadcast of batch b+1 (its own stream) overlaps batch b's kernels
        self.buffers = [torch.empty((self.w_max, 2), dtype=torch.int32, device=self.device) for _ in range(2)]
        self.buffer = self.buffers[0]
        self.m = 0
        self.nb = 0
        self.cuda = self.device.type == "cuda"
        self.exchange = self.world > 1 or force_exchange  # force: exercise the collective path at world 1 (tests)
        if self.cuda:
            self.comm = torch.cuda.Stream(device=self.device)
            self.consumed = [torch.cuda.Event() for _ in range(2)]

    def _engine_stream(self):
        ptr = getattr(self.engine, "stream_ptr", 0) if self.cuda else 0
        return torch.cuda.ExternalStream(ptr, device=self.device) if ptr else None

    def _exchange(self, fill, w):
        """Run fill(buf) -- the collective that leaves this batch in buf[:w] on every rank -- and return
        buf[:w] ready for the engine.  CUDA: on the comm stream, into the buffer the batch before last used
        (its kernels are done with it), and the engine stream waits for it; CPU (gloo): inline."""
        i = self.nb & 1
        buf = self.buffers[i]
        es = self._engine_stream()
        if not self.cuda or es is None:
            fill(buf)
            return buf[:w], None
        self.comm.wait_event(self.consumed[i])
        # rank 0's source tensor (or a host staging copy) may still be being produced on the caller's stream
        self.comm.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(self.comm):
            fill(buf)
            ready = torch.cuda.Event()
            ready.record(self.comm)
        es.wait_event(ready)
        return buf[:w], (es, i)

    def _push(self, batch, w, tok):
        eng_in = batch if not (self.device.type == "cpu") else batch.numpy().view("uint32")
        rc = self.engine.push_batch(eng_in)
        if tok is not None:
            es, i = tok
            self.consumed[i].record(es)
        if rc != 0:
            raise RuntimeError(f"push_batch failed on rank {self.rank}: {rc}")
        self.m += w
        self.nb += 1
        return rc

    def push_batch(self, edges, w: int | None = None):
        """Rank 0 passes the batch (a (w, 2) uint32/int32 tensor or array); the others pass None.  Unless
        every rank passes w, the batch size is broadcast first (a host synchronisation); then the edges are
        broadcast into a batch buffer and every rank updates its shard."""
        if not self.exchange:
            n = len(edges)
            if n == 0:
                return 0
            self.engine.push_batch(edges)
            self.m += n
            self.nb += 1
            return 0
        if w is None:
            n = torch.tensor([0 if edges is None else len(edges)], dtype=torch.int64, device=self.device)
            dist.broadcast(n, src=0, group=self.group)
            w = int(n.item())
        if w > self.w_max:
            raise ValueError("batch larger than w_max")
        if w == 0:
            return 0

        def fill(buf):
            if self.rank == 0:
                src = torch.as_tensor(edges) if not isinstance(edges, torch.Tensor) else edges
                buf[:w].copy_(src.view(torch.int32).reshape(w, 2), non_blocking=True)
            dist.broadcast(buf[:w], src=0, group=self.group)

        batch, tok = self._exchange(fill, w)
        return self._push(batch, w, tok)

    def push_batch_host(self, edges_host, w: int | None = None):
        """Host-fed batches: EVERY rank passes the same host batch; each copies only its
        1/G slice to its own GPU (its own PCIe link), then an all-gather assembles the batch on every GPU."""
        w = len(edges_host) if w is None else int(w)
        if w > self.w_max:
            raise ValueError("batch larger than w_max")
        if w == 0:
            return 0
        if not self.exchange:
            return self.push_batch(edges_host)
        per = -(-w // self.world)  # equal chunks for the all-gather; the last one padded
        if per * self.world > self.w_max:
            raise ValueError("w_max too small for the padded all-gather")
        src = torch.as_tensor(edges_host) if not isinstance(edges_host, torch.Tensor) else edges_host
        src = src.view(torch.int32).reshape(w, 2)
        lo, hi = self.rank * per, min(w, (self.rank + 1) * per)

        if getattr(self, "_slice", None) is None or self._slice.shape[0] < per:
            self._slice = torch.zeros((per, 2), dtype=torch.int32, device=self.device)

        def fill(buf):
            mine = self._slice[:per]
            if hi > lo:
                mine[: hi - lo].copy_(src[lo:hi], non_blocking=True)
            if hi - lo < per:
                mine[max(0, hi - lo):].zero_()
            dist.all_gather_into_tensor(buf[: per * self.world], mine, group=self.group)

        batch, tok = self._exchange(fill, w)
        return self._push(batch, w, tok)

    def closed_sum(self) -> int:
        """S over ALL ranks (exact integer all-reduce of the per-rank partial sums)."""
        s = torch.tensor([self.engine.closed_sum()], dtype=torch.int64, device=self.buffer.device)
        if self.world > 1:
            dist.all_reduce(s, op=dist.ReduceOp.SUM, group=self.group)
        return int(s.item())

    def estimate(self) -> float:
        """m * S / r as one fixed fp64 expression (reading R9) -- identical on every rank."""
        return float(self.m) * float(self.closed_sum()) / float(self.r)


class RankCounter:
    """The production multi-GPU path: this rank's shard behind tc_create_rank, the batch broadcast and the
    partial-sum all-reduce done by NCCL INSIDE the library (include/tc.h).  torch.distributed only
    bootstraps it (rank 0's 128-byte ncclUniqueId is broadcast over the default process group).

    push_batch(edges, w): rank 0 passes the batch (host array / tensor or a CUDA tensor on its device), the
    other ranks pass None; every rank passes the same w.  estimate() / closed_sum() are collective."""

    def __init__(self, r: int, seed: int, w_max: int, device=None, group=None):
        from . import TriangleCounter, nccl_unique_id
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        uid = bytearray(nccl_unique_id() if self.rank == 0 else bytes(128))
        if self.world > 1:
            t = torch.tensor(list(uid), dtype=torch.uint8,
                             device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
            dist.broadcast(t, src=0, group=group)
            uid = bytes(t.cpu().tolist())
        dev = torch.cuda.current_device() if device is None else int(torch.device(device).index or 0)
        self.engine = TriangleCounter.rank(r, seed, self.rank, self.world, bytes(uid), device=dev, w_max_hint=w_max)
        self.r, self.seed = int(r), int(seed)
        self.first, self.count = self.engine.first, self.engine.count
        assert (self.first, self.count) == shard(self.r, self.rank, self.world)

    def push_batch(self, edges, w: int | None = None):
        if edges is None:
            return self.engine.push_batch(None, w=int(w))
        return self.engine.push_batch(edges)

    def closed_sum(self) -> int:
        return self.engine.closed_sum()

    def estimate(self) -> float:
        return self.engine.estimate()
