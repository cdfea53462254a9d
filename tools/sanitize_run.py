"""A small workload that drives every kernel path of the library, for compute-sanitizer
(tests/test_sanitizers.py runs it under ONE tool per process): C1 batches, a hub stream through every
vertex-bucket path (hash, hub peeling, radix sort in shared and global memory, split partition), the
small-batch and the split per-step estimator passes, the event-driven mode, asynchronous and strict errors,
CUDA graphs, and a world-1 NCCL rank handle.  Exits non-zero if a result differs from the oracle."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    from gpu_common import assert_states_equal, oracle_run
    from paper_1308_2166_b200 import TriangleCounter
    from synth import er, rmat
    s1 = er(1000, 8000, 1)
    tc = TriangleCounter(1024, 42)
    for k in range(0, len(s1), 2048):
        tc.push_batch(s1[k:k + 2048])
    assert_states_equal(tc.state(), oracle_run(s1, 1024, 42, 2048).state(), "C1")
    hub = rmat(12, 16, 3)[:20000]
    for knobs in (dict(), dict(vbucket_cap=1, vbucket_sort_cap=1), dict(vbucket_cap=1), dict(vbucket_arcs=1),
                  dict(vbucket_arcs=8192, vbucket_cap=1), dict(small_batch=2), dict(split_kernels=1)):
        for graphs in (False, True):
            t = TriangleCounter(700, 5)
            t.tune(**knobs)
            t.set_graphs(graphs)
            t.set_async(graphs)
            for k in range(0, len(hub), 6000):
                t.push_batch(hub[k:k + 6000])
            assert t.sync() == 0
            assert_states_equal(t.state(), oracle_run(hub, 700, 5, 6000).state(), f"{knobs} graphs={graphs}")
    # the one-CTA index and the partitioned build at the same small batch size
    for si in (2, 1):
        t = TriangleCounter(900, 7)
        t.tune(small_index=si)
        for k in range(0, len(hub), 2000):
            t.push_batch(hub[k:k + 2000])
        assert_states_equal(t.state(), oracle_run(hub, 900, 7, 2000).state(), f"small_index={si}")
    # the event-driven mode: small (one-CTA) and partitioned index, strict and graphs + asynchronous errors
    from oracle.edc import EventOracleC
    for w, graphs, checked in ((2000, False, 0), (6000, True, 0), (333, True, 0), (2000, True, 1), (6000, False, 1)):
        t = TriangleCounter(800, 11)
        t.set_mode("event")
        t.tune(event_checked=checked)
        t.set_graphs(graphs)
        t.set_async(graphs)
        o = EventOracleC(800, 11)
        for k in range(0, len(hub), w):
            t.push_batch(hub[k:k + w])
            o.push_batch(hub[k:k + w], validate=False)
        assert t.sync() == 0
        assert_states_equal(t.state(), o.state(), f"event mode w={w}")
        assert t.closed_sum() == o.closed_sum()
    bad = np.array([[1, 2], [3, 3]], np.uint32)
    assert tc.push_batch(bad, check=False) != 0
    if os.environ.get("TC_SANITIZE_NCCL", "1") == "1":
        from paper_1308_2166_b200 import nccl_unique_id
        rk = TriangleCounter.rank(500, 9, 0, 1, nccl_unique_id(), device=0)
        for k in range(0, len(hub), 5000):
            rk.push_batch(hub[k:k + 5000])
        assert rk.closed_sum() == oracle_run(hub, 500, 9, 5000).closed_sum()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
