"""GPU parity: the CUDA path (through the C ABI) vs the oracle, bit for bit on every estimator field.

Sizes span several tiles (256-estimator blocks, 2048-arc sort chunks) with ragged tails; the full
BASELINE.json C2 size runs in the bench's launch configuration with sampled estimator shards checked
against the oracle and NBSI properties checked on every estimator.
"""
import numpy as np
import pytest

from gpu_common import FIELDS, assert_states_equal, check_properties, gpu_run, oracle_run
from synth import er, rmat

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - only on CPU boxes, where -m gpu is not run
    pytest.skip("no CUDA device", allow_module_level=True)


@pytest.fixture(scope="module", autouse=True)
def lib():
    import paper_1308_2166_b200 as pkg
    from paper_1308_2166_b200 import build
    build.build()
    return pkg.load_library()


def _compare(stream, r, seed, w, **kw):
    g = gpu_run(stream, r, seed, w, **kw)
    o = oracle_run(stream, r, seed, w, kw.get("first", 0), kw.get("count"))
    assert_states_equal(g.state(), o.state(), f"r={r} seed={seed} w={w}")
    assert g.closed_sum() == o.closed_sum()
    assert g.estimate() == o.estimate()
    assert g.counters() == o.counters()
    return g, o


def test_worked_example():
    A, B, C, D, E, F = range(6)
    old = [(C, E), (A, C), (A, F)]
    W = [(B, C), (C, D), (E, F), (B, D), (D, F)]
    s = np.array(old + W, dtype=np.uint32)
    for seed in range(8):
        g = gpu_run(s[:3], 300, seed, 3)
        g.push_batch(s[3:])
        o = oracle_run(s[:3], 300, seed, 3)
        o.push_batch(s[3:])
        assert_states_equal(g.state(), o.state())


@pytest.mark.parametrize("seed", range(6))
def test_tiny_random_batchings(seed):
    rnd = np.random.default_rng(seed)
    s = er(int(rnd.integers(8, 60)), int(rnd.integers(20, 150)), seed)
    for w in (1, 2, 3, 7, 16, 1000):
        _compare(s, int(rnd.integers(1, 700)), seed * 10 + w, w)


@pytest.mark.parametrize("seed", [42, 0, 7])
def test_C1_full(seed):
    s = er(1000, 20000, 1)
    _compare(s, 4096, seed, 2048)


def test_C1_per_batch_states():
    s = er(1000, 20000, 1)
    g = gpu_run(s[:0], 4096, 3, 2048)
    from oracle.indexed import IndexedOracle
    o = IndexedOracle(4096, 3)
    for k in range(0, len(s), 2048):
        g.push_batch(s[k:k + 2048])
        assert o.push_batch(s[k:k + 2048]) == 0
        assert_states_equal(g.state(), o.state(), f"after batch {k // 2048}")


def _hub_stream():
    """A star with 5000 leaves plus ER noise, deduplicated, random order and orientation."""
    rng = np.random.default_rng(5)
    leaves = rng.permutation(np.arange(1, 9000, dtype=np.uint32))[:5000]
    star = np.stack([np.zeros(5000, np.uint32), leaves], 1)
    noise = er(9000, 6000, 11)
    noise = noise[(noise[:, 0] != 0) & (noise[:, 1] != 0)]
    s = np.concatenate([star, noise])
    s = s[rng.permutation(len(s))]
    flip = rng.random(len(s)) < 0.5
    s[flip] = s[flip][:, ::-1]
    keys = np.sort(s, 1)
    _, uniq = np.unique(keys[:, 0].astype(np.uint64) << np.uint64(32) | keys[:, 1], return_index=True)
    return np.ascontiguousarray(s[np.sort(uniq)])


def test_hub_segments_multi_chunk():
    """The hub's vertex bucket (> 4096 arcs at the largest w) takes the chunked global-memory path."""
    s = _hub_stream()
    for w in (len(s), 4099, 700):
        _compare(s, 3000, 99 + w, w)


@pytest.mark.parametrize("knobs", [
    dict(vbucket_cap=1, vbucket_sort_cap=1),       # every bucket through the hub-peel kernel; deferred ones chunked
    dict(vbucket_cap=1),                           # every vertex bucket through the hub-peel kernel
    dict(vbucket_arcs=8192, vbucket_cap=1),        # hub-less buckets > 4096 arcs: radix sort in shared memory
    dict(vbucket_cap=37, vbucket_sort_cap=200),    # a mix of all paths
    dict(vbucket_arcs=16),                         # many buckets
    dict(vbucket_arcs=1),                          # 2^15 buckets: 4096 partition buckets split 8 ways (k_split)
    dict(vbucket_arcs=2, vbucket_cap=3),           # split + most sub-buckets through the large-bucket kernels
    dict(vbucket_arcs=1 << 30),                    # one vertex bucket
    dict(small_batch=1),                           # the full estimator pass even for small batches
    dict(small_batch=2),                           # the filtered small-batch pass even for large batches
    dict(small_index=1, small_batch=1),            # small batches through the partitioned build
    dict(small_index=2, split_kernels=1),          # one-CTA index + split estimator pass
    dict(pair_filter=2),                           # Step 3 behind the pair filter at every size
    dict(pair_filter=2, small_batch=2, vbucket_arcs=2),  # pair filter + filtered pass + split partition
    dict(small_index_arcs=16),                     # one-CTA index on its maximum of 256 CTAs
    dict(small_index_arcs=8192, small_batch=2),    # one-CTA index on a single CTA
])
def test_index_geometry_knobs(knobs):
    """Results never depend on the index geometry (tc_tune): bit-exact against the oracle.  Batches of at most
    4096 edges take the one-CTA index unless small_index=1, so the geometry knobs are also run with it off."""
    from paper_1308_2166_b200 import TriangleCounter
    s = _hub_stream()
    for w, extra in ((len(s), {}), (2500, {}), (2500, {"small_index": 1}), (1, {}), (1, {"small_index": 1})):
        ww = w if w > 1 else 1
        tc = TriangleCounter(1500, 5 + w)
        tc.tune(**{**knobs, **extra})
        n = len(s) if w > 1 else 300
        for k in range(0, n, ww):
            tc.push_batch(s[k:min(n, k + ww)])
        o = oracle_run(s[:n], 1500, 5 + w, ww)
        assert_states_equal(tc.state(), o.state(), f"{knobs} {extra} w={w}")


def test_device_pinned_pageable_inputs_agree():
    s = rmat(12, 16, 4)
    w = 5001
    a = gpu_run(s, 2000, 1, w).state()
    b = gpu_run(s, 2000, 1, w, device_input=True).state()
    assert_states_equal(a, b, "device vs pageable")
    from paper_1308_2166_b200 import TriangleCounter
    pinned = torch.from_numpy(s.view(np.int32)).pin_memory()
    tc = TriangleCounter(2000, 1)
    for k in range(0, len(s), w):
        tc.push_batch(pinned[k:k + w])
    assert_states_equal(a, tc.state(), "pinned vs pageable")
    # misaligned device pointer (odd edge offset): the scalar staging path
    d = torch.from_numpy(np.concatenate([np.zeros((1, 2), np.uint32), s]).view(np.int32)).cuda()
    tc2 = TriangleCounter(2000, 1)
    for k in range(0, len(s), w):
        tc2.push_batch(d[1 + k:1 + k + min(w, len(s) - k)])
    assert_states_equal(a, tc2.state(), "misaligned device")


def test_shards_equal_whole():
    s = rmat(11, 16, 6)
    whole = gpu_run(s, 3001, 8, 1500).state()
    parts = [gpu_run(s, 3001, 8, 1500, first=f, count=c).state() for f, c in ((0, 1000), (1000, 1), (1001, 2000))]
    for f in FIELDS:
        np.testing.assert_array_equal(whole[f], np.concatenate([p[f] for p in parts]))


def test_errors_all_or_nothing_and_async():
    from paper_1308_2166_b200 import TriangleCounter
    from paper_1308_2166_b200._lib import TC_EDUP, TC_EINVAL, TC_ESELFLOOP, TC_ESTATE
    s = er(50, 400, 3)
    tc = TriangleCounter(500, 2)
    tc.push_batch(s[:200])
    before = tc.state()
    assert tc.push_batch(s[:0], check=False) == 0
    cases = [
        (np.concatenate([s[200:220], [[5, 5]]]), TC_ESELFLOOP),
        (np.concatenate([s[200:220], s[205:206, ::-1]]), TC_EDUP),
        (np.concatenate([[[1, 0xFFFFFFFF]], s[200:220]]), TC_EINVAL),
        (np.array([[4, 4], [0xFFFFFFFF, 2], [1, 2], [2, 1]]), TC_EINVAL),
        (np.array([[4, 4], [1, 2], [2, 1]]), TC_ESELFLOOP),
    ]
    for W, code in cases:
        assert tc.push_batch(np.ascontiguousarray(W, dtype=np.uint32), check=False) == code
        assert_states_equal(before, tc.state(), f"after rejected batch {code}")
        assert tc.counters() == (200, 1)
    tc.push_batch(s[200:])
    assert_states_equal(tc.state(), oracle_run(s, 500, 2, 200).state(), "after recovery")
    # asynchronous errors: sticky, reported at the next synchronising call, state kept
    tc2 = TriangleCounter(500, 2)
    tc2.set_async(True)
    tc2.push_batch(s[:200])
    good = oracle_run(s[:200], 500, 2, 200).state()
    assert tc2.push_batch(np.array([[3, 3]], np.uint32), check=False) == 0
    assert tc2.push_batch(s[200:], check=False) == 0
    assert tc2.sync() == TC_ESELFLOOP
    assert tc2.push_batch(s[200:], check=False) == TC_ESTATE
    assert_states_equal(good, tc2.state(), "async poisoned")


def test_mom_and_group_sums():
    from oracle import nbsi
    s = er(300, 5000, 2)
    g, o = _compare(s, 3000, 12, 777)
    st = o.state()
    m = len(s)
    for groups in (1, 2, 7, 64, 3000):
        assert g.estimate_mom(groups) == nbsi.median_of_means(st, m, groups)
        n = 3000
        ref = [sum(int(st["c"][i]) for i in range(gg * n // groups, (gg + 1) * n // groups) if st["closed"][i])
               for gg in range(groups)]
        assert g.group_sums(groups).tolist() == ref


def test_graph_and_plain_launches_agree():
    """The CUDA-graph launch path (default) and plain stream launches give identical states."""
    from paper_1308_2166_b200 import TriangleCounter
    s = rmat(13, 16, 9)
    out = []
    for graphs in (True, False):
        tc = TriangleCounter(5000, 77)
        tc.set_graphs(graphs)
        tc.set_async(True)
        k = 0
        for w in (4096, 4096, 333, 4096, 1, 7000, 4096):
            tc.push_batch(s[k:k + w])
            k += w
        assert tc.sync() == 0
        out.append(tc.state())
        if graphs:  # one capture per batch shape (4), the index growth at 7000 drops them once
            assert 4 <= tc.graph_captures() <= 6
    assert_states_equal(out[0], out[1], "graph vs plain")
    from oracle.indexed import IndexedOracle
    o = IndexedOracle(5000, 77)
    k = 0
    for w in (4096, 4096, 333, 4096, 1, 7000, 4096):
        assert o.push_batch(s[k:k + w]) == 0
        k += w
    assert_states_equal(out[0], o.state(), "graph vs oracle")


def test_async_host_uploads_and_closed_sum_async():
    """Host batches in asynchronous mode go through the two alternating staging buffers on the copy stream
    (the upload of batch b+1 overlaps batch b's kernels); mixing pinned, pageable and device batches, with
    and without graphs, must leave the oracle's state, and tc_closed_sum_async must return every batch's S."""
    from paper_1308_2166_b200 import TriangleCounter
    from oracle.indexed import IndexedOracle
    s = rmat(13, 16, 5)
    ws = [3000, 5000, 1, 4096, 2500, 6000, 4096, 4096, 777]
    pinned = torch.from_numpy(s.view(np.int32)).pin_memory()
    dev = torch.from_numpy(s.view(np.int32)).cuda()
    o = IndexedOracle(3000, 21)
    ref_S = []
    k = 0
    for w in ws:
        assert o.push_batch(s[k:k + w]) == 0
        ref_S.append(o.closed_sum())
        k += w
    for graphs in (True, False):
        tc = TriangleCounter(3000, 21)
        tc.set_async(True)
        tc.set_graphs(graphs)
        Sbuf = torch.zeros(len(ws), dtype=torch.int64).pin_memory()
        k = 0
        for i, w in enumerate(ws):
            src = (pinned, s, pinned, dev)[i % 4]
            tc.push_batch(src[k:k + w])
            tc.closed_sum_async(Sbuf, i)
            k += w
        assert tc.sync() == 0
        assert Sbuf.tolist() == ref_S
        assert_states_equal(tc.state(), o.state(), f"async uploads graphs={graphs}")


@pytest.mark.parametrize("mode", [1, 2])
def test_small_batch_pass_long_stream(mode):
    """Many small batches through many estimators (the regime of the filtered pass): the
    filtered pass (mode 2, also the default at these sizes) and the full pass (mode 1) both equal the
    oracle bit for bit, including the closed sums after every batch."""
    from paper_1308_2166_b200 import TriangleCounter
    s = rmat(12, 16, 8)[:30000]
    r, w = 20000, 512
    tc = TriangleCounter(r, 3)
    tc.tune(small_batch=mode)
    tc.set_async(True)
    Sbuf = torch.zeros(len(range(0, len(s), w)), dtype=torch.int64).pin_memory()
    for i, k in enumerate(range(0, len(s), w)):
        tc.push_batch(s[k:k + w])
        tc.closed_sum_async(Sbuf, i)
    assert tc.sync() == 0
    from oracle.indexed import IndexedOracle
    o = IndexedOracle(r, 3)
    ref = []
    for k in range(0, len(s), w):
        assert o.push_batch(s[k:k + w]) == 0
        ref.append(o.closed_sum())
    assert Sbuf.tolist() == ref
    assert_states_equal(tc.state(), o.state(), f"small-batch mode {mode}")


def test_reset_limits_and_poison_recovery():
    """tc_reset restores the just-created state (also clearing a poisoned handle); oversized calls are
    rejected before touching memory (include/tc.h)."""
    import ctypes as C
    from paper_1308_2166_b200 import TriangleCounter, load_library
    from paper_1308_2166_b200._lib import TC_EINVAL, TC_ESELFLOOP
    s = rmat(11, 16, 12)
    tc = TriangleCounter(2500, 8)
    for k in range(0, len(s) // 2, 3000):
        tc.push_batch(s[k:k + 3000])
    tc.reset()
    assert tc.counters() == (0, 0) and tc.estimate() == 0.0
    for k in range(0, len(s), 3000):
        tc.push_batch(s[k:k + 3000])
    assert_states_equal(tc.state(), oracle_run(s, 2500, 8, 3000).state(), "after reset")
    # poisoned (asynchronous error) -> reset -> usable again
    tc.set_async(True)
    tc.push_batch(np.array([[9, 9]], np.uint32), check=False)
    assert tc.sync() == TC_ESELFLOOP
    tc.reset()
    tc.set_async(False)
    for k in range(0, len(s), 3000):
        tc.push_batch(s[k:k + 3000])
    assert_states_equal(tc.state(), oracle_run(s, 2500, 8, 3000).state(), "after poisoned reset")
    # w > 2^28 and m >= 2^31 are rejected up front
    assert tc.push_batch_ptr(s.ctypes.data, (1 << 28) + 1) == TC_EINVAL
    tau, ms = C.c_uint64(), C.c_double()
    assert load_library().tc_exact_triangles(C.c_void_p(s.ctypes.data), 1 << 31, C.byref(tau), C.byref(ms)) == TC_EINVAL


def test_C1_many_seeds_parity_and_statistics():
    """C1 over 1000 estimator seeds: every seed's final state equals the oracle's (compared by
    closed sum and a state digest), and the mean GPU estimate lies within 4 sigma of the exact tau, sigma
    from the closed-form variance Var X = m * sum_t C(t) - tau^2 (Claim discovery-prob)
    over r * seeds independent estimators."""
    import hashlib
    from oracle import exact
    from oracle.indexed import IndexedOracle
    from paper_1308_2166_b200 import TriangleCounter
    s = er(1000, 20000, 1)
    r, w, seeds = 4096, 2048, 1000
    dev = torch.from_numpy(s.view(np.int32)).cuda()
    ests = []

    def digest(st):
        h = hashlib.sha1()
        for f in FIELDS:
            h.update(np.ascontiguousarray(st[f]).tobytes())
        return h.hexdigest()

    for seed in range(seeds):
        g = TriangleCounter(r, 1000 + seed, w_max_hint=w)
        for k in range(0, len(s), w):
            g.push_batch(dev[k:k + w])
        o = IndexedOracle(r, 1000 + seed)
        for k in range(0, len(s), w):
            assert o.push_batch(s[k:k + w]) == 0
        assert g.closed_sum() == o.closed_sum(), seed
        if seed % 50 == 0:
            assert digest(g.state()) == digest(o.state()), seed
        ests.append(g.estimate())
        g.close()
    tau, sumC, m = exact.moments(s)
    var_x = m * sumC - tau * tau
    sigma = (var_x / (r * seeds)) ** 0.5
    assert abs(float(np.mean(ests)) - tau) <= 4 * sigma, (np.mean(ests), tau, sigma)


def test_checkpoint_resume():
    """tc_get_state / tc_counters -> tc_set_state / tc_set_counters on a fresh handle resumes the stream
    bit-exactly (the next push draws with the restored batch index); invalid snapshots are rejected
    without effect."""
    from paper_1308_2166_b200 import TCError, TriangleCounter
    s = rmat(12, 16, 21)
    r, w = 3000, 2500
    ref = oracle_run(s, r, 4, w)
    a = TriangleCounter(r, 4)
    half = (len(s) // w // 2) * w
    for k in range(0, half, w):
        a.push_batch(s[k:k + w])
    snap, (m, b) = a.state(), a.counters()
    a.close()
    c = TriangleCounter(r, 4)
    c.set_state(snap)
    c.set_counters(m, b)
    assert c.closed_sum() == int(snap["c"][snap["closed"] == 1].astype(np.int64).sum())
    for k in range(half, len(s), w):
        c.push_batch(s[k:k + w])
    assert_states_equal(c.state(), ref.state(), "resumed")
    assert c.estimate() == ref.estimate() and c.counters() == ref.counters()
    bad = {f: v.copy() for f, v in snap.items()}
    bad["r1"][5] = bad["r1"][5][::-1]  # lo > hi
    before = c.state()
    with pytest.raises(TCError):
        c.set_state(bad)
    assert_states_equal(c.state(), before, "rejected snapshot")
    with pytest.raises(TCError):
        c.set_counters(0, 3)


def _shuffled(edges, seed):
    rng = np.random.default_rng(seed)
    e = np.asarray(edges, dtype=np.uint32)
    e = e[rng.permutation(len(e))]
    flip = rng.random(len(e)) < 0.5
    e[flip] = e[flip][:, ::-1]
    return np.ascontiguousarray(e)


@pytest.mark.parametrize("kind", ["star", "path", "complete", "bipartite", "two_hubs"])
def test_degenerate_graphs(kind):
    """Degenerate shapes of the method: a star (one vertex in every edge: a single hub segment, no
    triangle), a path (no wedge closes), a dense complete graph, a bipartite graph (wedges, no triangle),
    and two hubs joined to every other vertex (triangles only through the hub edge)."""
    if kind == "star":
        g = [(0, i) for i in range(1, 20000)]
    elif kind == "path":
        g = [(i, i + 1) for i in range(20000)]
    elif kind == "complete":
        g = [(a, b) for a in range(160) for b in range(a + 1, 160)]
    elif kind == "bipartite":
        g = [(a, 1000 + b) for a in range(100) for b in range(150)]
    else:
        g = [(0, 1)] + [(h, i) for h in (0, 1) for i in range(2, 9000)]
    s = _shuffled(g, 3)
    for w in (len(s), 4096, 777):
        _compare(s, 5000, 31 + w, w)


@pytest.mark.parametrize("case", range(64))
def test_fuzz_configurations(case):
    """Random graph, r, batch-size sequence, index knobs, launch mode and input placement per case; the
    CUDA path must equal the oracle bit for bit after every run."""
    from paper_1308_2166_b200 import TriangleCounter
    rng = np.random.default_rng(1000 + case)
    if rng.random() < 0.5:
        s = rmat(int(rng.integers(8, 13)), int(rng.integers(4, 17)), int(rng.integers(1, 99)))
    else:
        n = int(rng.integers(30, 3000))
        s = er(n, int(rng.integers(1, min(30000, n * (n - 1) // 2))), int(rng.integers(1, 99)))
    r = int(rng.choice([1, 2, 31, 257, 1000, 4096, 30000]))
    seed = int(rng.integers(0, 2**63))
    sizes, k = [], 0
    while k < len(s):
        w = int(rng.choice([1, 2, 7, 100, 1000, 4096, 5000, 20000]))
        sizes.append(min(w, len(s) - k))
        k += sizes[-1]
    tc = TriangleCounter(r, seed)
    knobs = {}
    if rng.random() < 0.4:
        knobs["small_batch"] = int(rng.integers(0, 3))
    if rng.random() < 0.3:
        knobs["vbucket_arcs"] = int(rng.choice([1, 16, 256, 4096]))
    if rng.random() < 0.3:
        knobs["vbucket_cap"] = int(rng.choice([1, 64, 2048]))
    if rng.random() < 0.3:
        knobs["small_index"] = int(rng.integers(0, 3))
    if knobs:
        tc.tune(**knobs)
    tc.set_graphs(bool(rng.random() < 0.5))
    tc.set_async(bool(rng.random() < 0.5))
    place = rng.integers(0, 3)
    src = {0: s, 1: torch.from_numpy(s.view(np.int32)).pin_memory(), 2: torch.from_numpy(s.view(np.int32)).cuda()}[int(place)]
    k = 0
    for w in sizes:
        tc.push_batch(src[k:k + w])
        k += w
    assert tc.sync() == 0
    from oracle.indexed import IndexedOracle
    o = IndexedOracle(r, seed)
    k = 0
    for w in sizes:
        assert o.push_batch(s[k:k + w]) == 0
        k += w
    assert_states_equal(tc.state(), o.state(), f"fuzz case {case} r={r} knobs={knobs} place={place}")
    assert tc.closed_sum() == o.closed_sum() and tc.counters() == o.counters()


def test_graph_relaunch_steady_stream():
    """A stream of equal batches captures ONE graph and relaunches it (per-batch values through the device
    descriptor); the ragged last batch adds one more shape.  States equal the oracle's."""
    from paper_1308_2166_b200 import TriangleCounter
    s = rmat(13, 16, 12)
    tc = TriangleCounter(4000, 6, w_max_hint=3000)
    tc.set_graphs(True)
    tc.set_async(True)
    for k in range(0, len(s), 3000):
        tc.push_batch(s[k:k + 3000])
    assert tc.sync() == 0
    assert tc.graph_captures() == (1 if len(s) % 3000 == 0 else 2)
    assert_states_equal(tc.state(), oracle_run(s, 4000, 6, 3000).state(), "graph relaunch")


@pytest.mark.parametrize("graphs", [False, True])
def test_pair_filter_mixed_sizes(graphs):
    """Step 3 behind the pair filter (tc_tune pair_filter=2): the two filters alternate by batch parity and k_count
    zeroes the next one, so batches of changing size, one-CTA-index batches (no filter) in between and a
    rejected batch must all leave the oracle's exact state."""
    from paper_1308_2166_b200 import TCError, TriangleCounter
    s = rmat(14, 12, 77)
    sizes = [9000, 300, 12000, 1, 7000, 5000, 4097, 20000, 2, 15000]
    tc = TriangleCounter(3000, 21)
    tc.tune(pair_filter=2)
    tc.set_graphs(graphs)
    o_bounds, k = [], 0
    for i, w in enumerate(sizes * 3):
        if k >= len(s):
            break
        if i == 7:  # a rejected batch (self-loop) changes nothing
            bad = np.array(s[k:k + 5000])
            bad[17] = [bad[17][0], bad[17][0]]
            with pytest.raises(TCError):
                tc.push_batch(bad)
        tc.push_batch(s[k:k + w])
        o_bounds.append((k, min(len(s), k + w)))
        k += w
    from oracle.indexed import IndexedOracle
    o = IndexedOracle(3000, 21, 0, None)
    for a, b in o_bounds:
        assert o.push_batch(s[a:b]) == 0
    assert_states_equal(tc.state(), o.state(), f"pair filter, graphs={graphs}")
