"""GPU tests of the C ABI's contract beyond the steady-state path: the device RNG functions against the
oracle's (including Lemire's rejection loop), asynchronous-error bookkeeping, checkpoint validation, the
library's m limit, and stream ordering of device inputs."""
import numpy as np
import pytest

from gpu_common import assert_states_equal, oracle_run
from synth import er, rmat

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)


@pytest.fixture(scope="module", autouse=True)
def lib():
    import paper_1308_2166_b200 as pkg
    from paper_1308_2166_b200 import build
    build.build()
    return pkg.load_library()


def test_device_lemire_matches_oracle_including_rejections():
    """philox.cuh::bounded (the estimator pass's draw, readings R7/R8) == oracle/indexed.c's Lemire on
    random inputs and on inputs that force the rejection loop: n = 3, x = 0 (rejected once at least),
    n = 2^63 + 1 with x = 2 (low64(x n) = 2 < threshold 2^63 - 1; each retry is rejected w.p. ~1/2)."""
    from oracle import indexed
    from paper_1308_2166_b200 import test_draws
    g = np.random.default_rng(3)
    k = 4000
    n = g.integers(1, 2**63, size=k, dtype=np.uint64)
    n[:500] = g.integers(1, 1000, size=500, dtype=np.uint64)
    x = g.integers(0, 2**63, size=k, dtype=np.uint64) * np.uint64(2) + g.integers(0, 2, size=k, dtype=np.uint64)
    ids = g.integers(0, 2**40, size=k, dtype=np.uint64)
    b = g.integers(0, 2**31, size=k, dtype=np.uint64).astype(np.uint32)
    base = np.where(g.random(k) < 0.5, 0x10000, 0x20000).astype(np.uint32)
    forced = [(3, 0), (2**63 + 1, 2), (2**63 + 1, 0), (5, 0), (2**64 - 1, 0), (2**64 - 1, 1)]
    for t, (nn, xx) in enumerate(forced):
        n[t], x[t] = nn, xx
    seed = 0x123456789ABCDEF
    got = test_draws(n, x, ids, b, base, seed)
    L = indexed.lib()
    for t in range(k):
        want = L.orc_lemire_words(int(n[t]), int(x[t]), seed, int(ids[t]), int(b[t]), int(base[t]))
        assert int(got[t]) == want, (t, int(n[t]), int(x[t]))
    # the forced cases really took the retry path (the first word alone would give another value or be rejected)
    for t, (nn, xx) in enumerate(forced[:2]):
        assert (xx * nn) % 2**64 < (2**64 - nn) % nn
        assert int(got[t]) < nn


def test_device_philox_matches_oracle():
    from oracle import rng
    from paper_1308_2166_b200 import test_philox
    g = np.random.default_rng(8)
    ctr = g.integers(0, 2**32, size=(1000, 4), dtype=np.uint64).astype(np.uint32)
    key = g.integers(0, 2**32, size=(1000, 2), dtype=np.uint64).astype(np.uint32)
    ctr[0] = 0
    key[0] = 0
    out = test_philox(ctr, key)
    for t in range(len(ctr)):
        assert tuple(int(v) for v in out[t]) == rng.philox4x32_10(tuple(ctr[t]), tuple(key[t]))


def test_async_error_survives_index_growth_and_counters_roll_back():
    """a rejected asynchronous batch followed by a LARGER batch (index reallocation) must still
    be reported, and m / the batch count go back to the last accepted batch (tc_counters settles)."""
    from paper_1308_2166_b200 import TriangleCounter
    from paper_1308_2166_b200._lib import TC_ESELFLOOP, TC_ESTATE
    s = er(300, 6000, 4)
    tc = TriangleCounter(700, 6)
    tc.set_async(True)
    tc.push_batch(s[:200])
    tc.push_batch(s[200:400])
    assert tc.push_batch(np.array([[3, 3], [1, 2]], np.uint32), check=False) == 0  # enqueued; bad
    tc.push_batch(s[400:450], check=False)  # skipped on the device (sticky error)
    rc = tc.push_batch(s[450:5450], check=False)  # w above the index capacity: grows -> must report
    assert rc == TC_ESELFLOOP
    assert tc.push_batch(s[450:500], check=False) == TC_ESTATE
    assert tc.counters() == (400, 2)
    assert_states_equal(tc.state(), oracle_run(s[:400], 700, 6, 200).state(), "rolled back")
    # checkpoint taken from the poisoned handle resumes exactly on a fresh handle
    snap, (m, b) = tc.state(), tc.counters()
    c = TriangleCounter(700, 6)
    c.set_state(snap)
    c.set_counters(m, b)
    c.push_batch(s[400:1400])
    ref = oracle_run(s[:400], 700, 6, 200)
    assert ref.push_batch(s[400:1400]) == 0
    assert_states_equal(c.state(), ref.state(), "resumed from poisoned checkpoint")
    assert c.closed_sum() == ref.closed_sum()


def test_reset_right_after_async_failure():
    """tc_reset on a handle whose asynchronous failure was not yet reported must clear it."""
    from paper_1308_2166_b200 import TriangleCounter
    s = er(100, 1000, 2)
    tc = TriangleCounter(300, 1)
    tc.set_async(True)
    tc.push_batch(s[:300])
    tc.push_batch(np.array([[7, 7]], np.uint32), check=False)
    tc.reset()  # no sync() first
    assert tc.counters() == (0, 0)
    for k in range(0, len(s), 250):
        tc.push_batch(s[k:k + 250])
    assert tc.sync() == 0
    assert_states_equal(tc.state(), oracle_run(s, 300, 1, 250).state(), "after reset")


def test_async_failure_then_more_batches_counts():
    """m and b after a mid-pipeline rejection: several good batches, a bad one, more good ones, all
    enqueued before the sync; the state and the counters are those after the last good batch before it."""
    from paper_1308_2166_b200 import TriangleCounter
    from paper_1308_2166_b200._lib import TC_EDUP
    s = rmat(11, 16, 3)
    tc = TriangleCounter(2000, 9)
    tc.set_async(True)
    tc.set_graphs(True)
    for k in range(0, 3000, 1000):
        tc.push_batch(s[k:k + 1000])
    dup = np.concatenate([s[3000:3100], s[3050:3051, ::-1]])
    tc.push_batch(np.ascontiguousarray(dup), check=False)
    for k in range(3100, 6000, 1000):
        tc.push_batch(s[k:k + 1000], check=False)
    assert tc.sync() == TC_EDUP
    assert tc.counters() == (3000, 3)
    ref = oracle_run(s[:3000], 2000, 9, 1000)
    assert_states_equal(tc.state(), ref.state(), "after mid-pipeline rejection")
    tc.reset()


def test_set_state_rejects_nbsi_violations():
    """checkpoints that break the invariants the estimator pass relies on are rejected."""
    from paper_1308_2166_b200 import TCError, TriangleCounter
    s = er(60, 800, 5)
    tc = TriangleCounter(50, 3)
    tc.push_batch(s)
    good = tc.state()
    i = int(np.nonzero(good["c"] > 0)[0][0])
    E = 0xFFFFFFFF

    def mutated(**kw):
        st = {f: v.copy() for f, v in good.items()}
        for f, v in kw.items():
            st[f][i] = v
        return st

    r1 = good["r1"][i]
    bad = [
        mutated(c=0),                                                       # f2 present, chi = 0
        mutated(r2=[E, E], p2=2**64 - 1),                                    # f2 empty, chi > 0
        mutated(r2=[max(r1) + 1, max(r1) + 2]),                              # f2 not adjacent to f1
        mutated(r2=list(r1)),                                                # f2 == f1 (two shared endpoints)
        mutated(p2=int(good["p1"][i])),                                      # p2 not after p1
        mutated(r1=[E, E], p1=2**64 - 1),                                    # empty f1 with f2 / chi
    ]
    for st in bad:
        with pytest.raises(TCError):
            tc.set_state(st)
        assert_states_equal(tc.state(), good, "rejected checkpoint")
    tc.set_state(good)


def test_library_m_limit():
    """The library's documented limit (include/tc.h, DESIGN R13): m may not pass 2^31 - 1 (32-bit device
    positions); such a batch is rejected with TC_EOVERFLOW and nothing changes."""
    from paper_1308_2166_b200 import TriangleCounter
    from paper_1308_2166_b200._lib import TC_EOVERFLOW
    M = (1 << 31) - 10
    for async_ in (False, True):
        tc = TriangleCounter(100, 1)
        tc.set_async(async_)
        tc.set_counters(M, 1)
        before = tc.state()
        W = np.array([[2 * k, 2 * k + 1] for k in range(20)], np.uint32)
        assert tc.push_batch(W, check=False) == TC_EOVERFLOW
        assert tc.counters() == (M, 1)
        assert_states_equal(tc.state(), before, "m limit")
        assert tc.push_batch(W[:9], check=False) == 0
        assert tc.sync() == 0 and tc.counters() == (M + 9, 2)


def test_device_input_produced_on_another_stream():
    """A CUDA batch still being written on torch's current stream when push_batch is called: the engine's
    stream waits for it (tc_push_batch_after), in strict and asynchronous mode."""
    from paper_1308_2166_b200 import TriangleCounter
    s = rmat(12, 16, 7)
    w = 4000
    host = torch.from_numpy(s.view(np.int32)).pin_memory()
    ref = oracle_run(s, 1500, 2, w)
    for async_ in (False, True):
        tc = TriangleCounter(1500, 2)
        tc.set_async(async_)
        side = torch.cuda.Stream()
        bufs = [torch.empty((w, 2), dtype=torch.int32, device="cuda") for _ in range(3)]
        with torch.cuda.stream(side):
            for i, k in enumerate(range(0, len(s), w)):
                buf = bufs[i % 3][: min(w, len(s) - k)]
                torch.cuda._sleep(2_000_000)  # the copy lands well after push_batch is called
                buf.copy_(host[k:k + w], non_blocking=True)
                tc.push_batch(buf)
                # the buffer is reused 3 pushes later: wait until the engine is done with it
                ev = torch.cuda.Event()
                ev.record(torch.cuda.ExternalStream(tc.stream_ptr))
                side.wait_event(ev)
        assert tc.sync() == 0
        assert_states_equal(tc.state(), ref.state(), f"producer stream async={async_}")
