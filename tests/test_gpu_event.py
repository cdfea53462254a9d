"""GPU parity of the event-driven mode (tc_set_mode TC_MODE_EVENT, reading R17)
against oracle/ed.c (pinned to the plain per-edge oracle oracle/ed.py, itself pinned by exact enumeration):
every estimator, every field (r1, p1, r2, p2, chi, closed, J, K, ev), after every batch of random batchings, on
ER / R-MAT / C1 / C5-prefix streams; batch invariance on the GPU; the rejection paths; the vertex-table growth and
watch-pool rebuild paths; NBSI properties at size."""
import numpy as np
import pytest

from gpu_common import assert_states_equal, check_properties

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


def event_counter(r, seed, first=0, count=None, graphs=False, async_=False, w_max_hint=0, checked=False):
    from paper_1308_2166_b200 import TriangleCounter
    tc = TriangleCounter(r, seed, first=first, count=count, w_max_hint=w_max_hint)
    tc.set_mode("event")
    if checked:  # the four-kernel path that checks the degree limit first (else only past m + w > 2^30 - 1)
        tc.tune(event_checked=1)
    tc.set_graphs(graphs)
    tc.set_async(async_)
    return tc


def oracle(r, seed, first=0, count=None):
    from oracle.edc import EventOracleC
    return EventOracleC(r, seed, first, count)


def compare(tc, o, where):
    st, ost = tc.state(), o.state()
    assert_states_equal(st, ost, where)
    ev = tc.event_state()
    for f in ("J", "K", "ev"):
        if not np.array_equal(ev[f], ost[f].astype(np.uint32)):
            i = int(np.nonzero(ev[f] != ost[f].astype(np.uint32))[0][0])
            raise AssertionError(f"{where}: {f} differs (first at {i}: {ev[f][i]} vs {ost[f][i]})")
    assert tc.closed_sum() == o.closed_sum(), where
    return st


def _batchings(rng, m, sizes):
    out, k = [], 0
    while k < m:
        w = int(rng.choice(sizes))
        out.append((k, min(m, k + w)))
        k += w
    return out


@pytest.mark.parametrize("case", range(6))
def test_every_batch_random(case):
    from synth import er, rmat
    rng = np.random.default_rng(case)
    s = er(300, 6000, case) if case % 2 == 0 else rmat(11, 4, case)[:6000]
    s = np.ascontiguousarray(s, dtype=np.uint32)
    r = [1, 37, 2000, 5000][case % 4]
    graphs, async_ = case % 3 == 1, case % 3 == 2
    tc = event_counter(r, 100 + case, graphs=graphs, async_=async_, checked=case >= 3)
    if case in (2, 5):  # the one-CTA index on more CTAs (results do not depend on the geometry)
        tc.tune(small_index_arcs=64 if case == 2 else 128)
    o = oracle(r, 100 + case)
    for lo, hi in _batchings(rng, len(s), [1, 7, 64, 500, 1500, 4096]):
        tc.push_batch(s[lo:hi])
        assert o.push_batch(s[lo:hi], validate=False) == 0
        if async_:
            assert tc.sync() == 0
        compare(tc, o, f"case {case} after {hi} edges")
    assert tc.estimate() == o.estimate()


def test_batch_invariance_gpu():
    """The event mode's state after a prefix does not depend on how it was batched (one GPU run per batching)."""
    from synth import rmat
    s = np.ascontiguousarray(rmat(12, 8, 3)[:30000], dtype=np.uint32)
    states = []
    for sizes in ([30000], [1000], [4096], [17, 999, 5000]):
        tc = event_counter(3000, 5)
        rng = np.random.default_rng(len(sizes))
        for lo, hi in _batchings(rng, len(s), sizes):
            tc.push_batch(s[lo:hi])
        states.append((tc.state(), tc.event_state(), tc.closed_sum()))
    for st, ev, S in states[1:]:
        assert_states_equal(st, states[0][0], "batch invariance")
        for f in ev:
            assert np.array_equal(ev[f], states[0][1][f]), f
        assert S == states[0][2]


def test_C1_and_watch_path_used():
    """C1 (configs[0]: ER n=1000, m=20000, r=4096, w=2048), graphs + async as in the bench."""
    from synth import config_stream
    s = config_stream("C1")
    tc = event_counter(4096, 42, graphs=True, async_=True, w_max_hint=2048)
    tc2 = event_counter(4096, 42, graphs=True, async_=True, w_max_hint=2048, checked=True)
    o = oracle(4096, 42)
    for k in range(0, len(s), 2048):
        tc.push_batch(s[k:k + 2048])
        tc2.push_batch(s[k:k + 2048])
        o.push_batch(s[k:k + 2048], validate=False)
    assert tc.sync() == 0 and tc2.sync() == 0
    st = compare(tc, o, "C1")
    compare(tc2, o, "C1 checked path")
    check_properties(s, st, len(s))
    cnt = tc.event_counters()
    nb = (len(s) + 2047) // 2048
    assert cnt["sweeps"] < nb, cnt  # later batches went through the watch lists
    assert cnt["visited"] < nb * 4096, cnt


@pytest.mark.parametrize("lw", [12, 16, 20])
def test_C5_prefix(lw):
    """C5 (R-MAT scale 22, r = 2^22) at w = 2^12 / 2^16 / 2^20: 2^21 edges (+ a ragged tail), every estimator."""
    from synth import config_stream
    s = config_stream("C5")
    w, r = 1 << lw, 1 << 22
    m = (1 << 21) + 777
    s = np.ascontiguousarray(s[:m])
    tc = event_counter(r, 9, graphs=True, async_=True, w_max_hint=w, checked=lw == 16)
    dev = torch.from_numpy(s.view(np.int32)).cuda()
    for k in range(0, m, w):
        tc.push_batch(dev[k:k + w])
    assert tc.sync() == 0
    o = oracle(r, 9)
    o.push_batch(s, validate=False)
    st = compare(tc, o, f"C5 prefix w=2^{lw}")
    check_properties(s, st, m)


def test_rejections_strict_and_async():
    from paper_1308_2166_b200._lib import TC_EDUP, TC_ESELFLOOP, TC_ESTATE
    from synth import er
    s = np.ascontiguousarray(er(200, 3000, 4), dtype=np.uint32)
    tc = event_counter(700, 3)
    o = oracle(700, 3)
    tc.push_batch(s[:1000])
    o.push_batch(s[:1000], validate=False)
    bad = np.ascontiguousarray(np.concatenate([s[1000:1100], s[1010:1011, ::-1]]))
    assert tc.push_batch(bad, check=False) == TC_EDUP
    loop = np.array([[5, 5]], np.uint32)
    assert tc.push_batch(np.concatenate([s[1000:1050], loop]), check=False) == TC_ESELFLOOP
    compare(tc, o, "after rejections")
    tc.push_batch(s[1000:3000])
    o.push_batch(s[1000:3000], validate=False)
    compare(tc, o, "after recovery")
    # asynchronous: the rejected batch poisons the handle; the state is that of the last accepted batch
    ta = event_counter(700, 3, async_=True)
    ta.push_batch(s[:1000])
    ta.push_batch(bad, check=False)
    ta.push_batch(s[1100:1200], check=False)
    assert ta.sync() == TC_EDUP
    oa = oracle(700, 3)
    oa.push_batch(s[:1000], validate=False)
    assert_states_equal(ta.state(), oa.state(), "async rejected")
    assert ta.push_batch(s[1200:1300], check=False) == TC_ESTATE
    ta.reset()
    ta.push_batch(s[:3000])
    ob = oracle(700, 3)
    ob.push_batch(s[:3000], validate=False)
    compare(ta, ob, "after reset")


def test_mode_rules():
    from paper_1308_2166_b200 import TriangleCounter
    from paper_1308_2166_b200._lib import TCError
    from synth import er
    s = np.ascontiguousarray(er(50, 300, 1), dtype=np.uint32)
    tc = TriangleCounter(100, 1)
    tc.push_batch(s[:100])
    with pytest.raises(TCError):
        tc.set_mode("event")  # only before the first batch
    tc.reset()
    tc.set_mode("event")
    tc.push_batch(s)
    st = tc.state()
    with pytest.raises(TCError):
        tc.set_state(st)
    with pytest.raises(TCError):
        tc.set_counters(300, 1)
    o = oracle(100, 1)
    o.push_batch(s, validate=False)
    compare(tc, o, "mode switch after reset")
    # group sums / median of means from the same state
    ost = o.state()
    for g in (1, 3, 100):
        want = np.zeros(g, np.uint64)
        for i in range(100):
            if ost["closed"][i]:
                want[((i + 1) * g + 99) // 100 - 1] += np.uint64(ost["c"][i])
        assert tc.group_sums(g).tolist() == want.tolist()


def test_vertex_table_growth_and_pool_rebuilds():
    """Many distinct vertices from a small start (vertex-table rehash), and a small r over a long stream (the
    watch pool passes its threshold: full-sweep rebuilds), both against the oracle."""
    from synth import er
    s = np.ascontiguousarray(er(60000, 120000, 8), dtype=np.uint32)
    tc = event_counter(48, 2)  # no hint: the vertex table starts at 32K slots
    o = oracle(48, 2)
    rng = np.random.default_rng(1)
    for lo, hi in _batchings(rng, len(s), [33, 200, 1024]):
        tc.push_batch(s[lo:hi])
        o.push_batch(s[lo:hi], validate=False)
    compare(tc, o, "growth + rebuilds")
    cnt = tc.event_counters()
    assert cnt["vertices"] == len(np.unique(s))
    assert cnt["sweeps"] >= 2, cnt


def test_rank_handle_world1_event_mode():
    from paper_1308_2166_b200 import TriangleCounter, nccl_unique_id
    from synth import rmat
    s = np.ascontiguousarray(rmat(12, 8, 4)[:20000], dtype=np.uint32)
    tc = TriangleCounter.rank(3000, 11, 0, 1, nccl_unique_id(), device=0, w_max_hint=2500)
    tc.set_mode("event")
    tc.set_graphs(True)
    for k in range(0, len(s), 2500):
        tc.push_batch(s[k:k + 2500])
    o = oracle(3000, 11)
    o.push_batch(s, validate=False)
    compare(tc, o, "rank handle")
    assert tc.estimate() == o.estimate()


def test_event_mode_group_handle_graphs_and_async_sums():
    """tc_create_ex (one device) in the event mode; one graph capture per batch shape; tc_closed_sum_async per
    batch equal to the oracle's S after that prefix; median of means from the oracle's state."""
    from paper_1308_2166_b200 import TriangleCounter
    from synth import rmat
    s = np.ascontiguousarray(rmat(12, 8, 21)[:24000], dtype=np.uint32)
    w, r = 3000, 2500
    tc = TriangleCounter.multi(r, 17, [0], strict=False, graphs=True, w_max_hint=w)
    tc.set_mode("event")
    solo = event_counter(r, 17, graphs=True, async_=True, w_max_hint=w)
    Sbuf = torch.zeros(16, dtype=torch.int64).pin_memory()
    o = oracle(r, 17)
    ref = []
    for i, k in enumerate(range(0, len(s), w)):
        tc.push_batch(s[k:k + w])
        solo.push_batch(s[k:k + w])
        solo.closed_sum_async(Sbuf, i)
        o.push_batch(s[k:k + w], validate=False)
        ref.append(o.closed_sum())
    assert tc.sync() == 0 and solo.sync() == 0
    assert Sbuf[: len(ref)].tolist() == ref
    assert solo.graph_captures() <= 2  # the full-sweep and watch batches share one shape
    compare(tc, o, "tc_create_ex(1) event mode")
    compare(solo, o, "solo event mode")
    ost = o.state()
    m = len(s)
    for g in (1, 5, 50):
        means = []
        for j in range(g):
            lo, hi = j * r // g, (j + 1) * r // g
            Sg = int(ost["c"][lo:hi][ost["closed"][lo:hi] == 1].astype(np.int64).sum())
            means.append(float(m) * float(Sg) / float(hi - lo))
        assert tc.estimate_mom(g) == sorted(means)[(g - 1) // 2]
