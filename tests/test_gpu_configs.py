"""GPU parity at the BASELINE.json configs' full sizes, in the bench's launch configuration (one CUDA graph
per push, asynchronous errors, the stream resident in device memory -- or, for C4, pinned host memory):
EVERY estimator compared field by field with the oracle (oracle/indexed.c on the host cores), plus the
NBSI properties (gpu_common.check_properties) and the aggregate against a naive fp64 sum.

* C2 (configs[1]): the whole 15.7M-edge stream, r = w = 2^20, three estimator seeds.
* C3 (configs[2]): the whole 117M-edge Chung-Lu stream, r = 2^22, w = 2^23 (14 batches).
* C5 (configs[4]): R-MAT scale 22, r = 2^22, at every sweep batch size w = 2^12 .. 2^24 (three batches -- two from
  2^22 on -- plus a ragged tail of the stream each).
* Vertex ids spread over the whole id range [0, 0xFFFFFFFE].
* C4 (configs[3]): R-MAT scale 26 (~1B edges) streamed from pinned host memory at w = 2^24 with r = 2^24
  estimators on one GPU: the first two batches plus a ragged tail (the oracle's cost bounds the prefix).
"""
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


def bench_mode_run(stream, r, seed, w, first=0, count=None, host=False):
    """The CUDA path as bench.py drives it: graphs + asynchronous errors, device-resident (or pinned host)
    stream, w_max_hint = w."""
    from paper_1308_2166_b200 import TriangleCounter
    tc = TriangleCounter(r, seed, first=first, count=count, w_max_hint=w)
    tc.set_graphs(True)
    tc.set_async(True)
    src = torch.from_numpy(np.ascontiguousarray(stream).view(np.int32))
    src = src.pin_memory() if host else src.cuda()
    for k in range(0, len(stream), w):
        tc.push_batch(src[k:k + w])
    assert tc.sync() == 0
    return tc


def oracle_full(stream, r, seed, w, first=0, count=None):
    from oracle.indexed import IndexedOracle
    o = IndexedOracle(r, seed, first, count)
    for k in range(0, len(stream), w):
        assert o.push_batch(stream[k:k + w]) == 0
    return o


def compare_full(stream, r, seed, w, where, host=False):
    g = bench_mode_run(stream, r, seed, w, host=host)
    o = oracle_full(stream, r, seed, w)
    st = g.state()
    assert_states_equal(st, o.state(), where)
    assert g.closed_sum() == o.closed_sum() and g.counters() == o.counters()
    assert g.estimate() == o.estimate()
    m = len(stream)
    X = np.where(st["closed"] == 1, st["c"].astype(np.float64) * m, 0.0)
    naive = float(np.sum(X / r))
    assert abs(g.estimate() - naive) <= 1e-12 * abs(naive), (g.estimate(), naive)
    return st


@pytest.fixture(scope="module")
def c5_stream():
    from synth import config_stream
    return config_stream("C5")


@pytest.mark.parametrize("seed", [42, 7, 1234567])
def test_C2_full_state(seed):
    from synth import config_stream
    s = config_stream("C2")
    st = compare_full(s, 1 << 20, seed, 1 << 20, f"C2 seed {seed}")
    if seed == 42:
        check_properties(s, st, len(s))


def test_C3_full_state():
    from synth import config_stream
    s = config_stream("C3")
    assert len(s) == 117_000_000
    compare_full(s, 1 << 22, 42, 1 << 23, "C3 full stream")


@pytest.mark.parametrize("lw", list(range(12, 25)))
def test_C5_sweep_full_state(c5_stream, lw):
    w, r = 1 << lw, 1 << 22
    nb = 3 if lw <= 21 else 2  # the oracle's single-threaded sort of 2w arcs bounds the largest batches
    s = c5_stream[: nb * w + 123]
    st = compare_full(s, r, 9, w, f"C5 w=2^{lw}")
    if lw in (12, 20, 24):
        check_properties(s, st, len(s))


def test_full_range_vertex_ids():
    """Vertex ids spread over [0, 0xFFFFFFFE] (both extremes used): hashing, normalisation and the
    reserved id's neighbours."""
    from synth import native
    s = native.rmat(16, 16, 11)
    g = np.random.default_rng(4)
    vals = np.unique(g.integers(2, 0xFFFFFFFD, size=70000, dtype=np.uint64))[: (1 << 16)]
    ids = g.permutation(vals)[: 1 << 16].astype(np.uint32)  # an injective relabelling of [0, 2^16)
    hubs = np.argsort(-np.bincount(s.ravel().astype(np.int64), minlength=1 << 16), kind="stable")[:4]
    ids[hubs] = [0, 0xFFFFFFFE, 1, 0xFFFFFFFD]  # the extremes go to the busiest vertices
    assert len(np.unique(ids)) == 1 << 16
    t = np.ascontiguousarray(ids[s])
    assert t.max() == 0xFFFFFFFE and t.min() == 0
    for w in (1 << 15, 3000):
        st = compare_full(t, 1 << 16, 5, w, f"full-range ids w={w}")
    check_properties(t, st, len(t))


def test_C4_pinned_host_prefix():
    """C4: the R-MAT scale-26 stream (~1B unique edges, generated natively), fed from PINNED HOST memory
    through tc_push_batch at w = 2^24 with r = 2^24 on one GPU (the 8-GPU config's whole estimator set):
    the first two batches and a ragged tail, every estimator against the oracle, NBSI properties on all."""
    from synth import config_stream
    full = config_stream("C4")
    assert len(full) > 900_000_000 and full.max() < (1 << 26)
    w, r = 1 << 24, 1 << 24
    s = np.ascontiguousarray(full[: 2 * w + 4321])
    del full
    st = compare_full(s, r, 3, w, "C4 pinned-host prefix", host=True)
    check_properties(s, st, len(s))
