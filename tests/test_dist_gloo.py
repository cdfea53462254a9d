"""The multi-GPU plumbing (paper_1308_2166_b200/dist.py) on CPU: world_size 2 over gloo.

Each rank owns a contiguous shard of the estimators; rank 0 broadcasts every batch; the exact partial sums
are all-reduced.  The per-rank engine here is the CPU oracle (test infrastructure), so the check is that
the distributed host logic -- sharding, batch broadcast, all-reduce, estimate -- reproduces one unsharded
run bit for bit (the RNG is keyed by global estimator id, reading R7).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1308_2166_b200.dist import ShardedCounter, shard
from synth import er

R, SEED, W = 777, 9, 700


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, host_feed=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.indexed import IndexedOracle
        full = er(300, 5000, 4)
        stream = full if (rank == 0 or host_feed) else None
        sc = ShardedCounter(R, SEED, W + world, device="cpu",
                            engine_factory=lambda r, s, f, c: IndexedOracle(r, s, f, c))
        nb = (5000 + W - 1) // W
        for k in range(nb):
            if host_feed:  # every rank holds the batch, uploads its slice, all-gather
                sc.push_batch_host(torch.from_numpy(stream[k * W:(k + 1) * W].view("int32")))
            else:
                sc.push_batch(stream[k * W:(k + 1) * W] if rank == 0 else None)
        q.put((rank, sc.first, sc.count, sc.engine.state(), sc.closed_sum(), sc.estimate(), sc.m))
    finally:
        dist.destroy_process_group()


def test_shard_bounds():
    for r in (1, 7, 4096, 1 << 20):
        for world in (1, 2, 3, 8):
            if world > r:
                continue
            parts = [shard(r, g, world) for g in range(world)]
            assert parts[0][0] == 0 and sum(c for _, c in parts) == r
            assert all(parts[g][0] + parts[g][1] == parts[g + 1][0] for g in range(world - 1))
    with pytest.raises(ValueError):
        shard(10, 2, 2)


@pytest.mark.parametrize("host_feed", [False, True])
def test_two_ranks_gloo_equal_unsharded(host_feed):
    """Batch broadcast from rank 0 (host_feed False) or per-rank slices + all-gather (True)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(g, world, port, q, host_feed)) for g in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle.indexed import IndexedOracle
    stream = er(300, 5000, 4)
    whole = IndexedOracle(R, SEED)
    for k in range(0, len(stream), W):
        assert whole.push_batch(stream[k:k + W]) == 0
    ref = whole.state()
    for f in ref:
        got = np.concatenate([r_[3][f] for r_ in res])
        assert np.array_equal(got, ref[f]), f
    assert res[0][1:3] == (0, R // 2) and res[1][1:3] == (R // 2, R - R // 2)
    for r_ in res:  # every rank reports the same all-reduced S and estimate as the unsharded oracle
        assert r_[4] == whole.closed_sum()
        assert r_[5] == whole.estimate()
        assert r_[6] == len(stream)
