"""Multi-GPU machinery inside the library (include/tc.h tc_create_rank / tc_nccl_unique_id), exercised through
the C ABI on the one GPU available: a world-1 NCCL communicator runs the real broadcast and all-reduce code
paths (ncclBroadcast of every batch on the comm stream, ncclAllReduce of S and of the group sums).  The states
and every aggregate must equal the oracle's and a plain handle's.  (NCCL refuses two ranks on one GPU, so
world > 1 runs only on a multi-GPU box; the sharding itself is covered by test_dist_gloo.py on CPU.)"""
import numpy as np
import pytest

from gpu_common import assert_states_equal, oracle_run
from synth import rmat

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


@pytest.mark.parametrize("async_", [False, True])
@pytest.mark.parametrize("graphs", [False, True])
def test_rank_handle_world1_matches_oracle(async_, graphs):
    from paper_1308_2166_b200 import TriangleCounter, nccl_unique_id
    s = rmat(13, 16, 4)
    r, w = 3000, 5000
    tc = TriangleCounter.rank(r, 11, 0, 1, nccl_unique_id(), device=0, w_max_hint=w)
    assert (tc.first, tc.count, tc.rank_id, tc.world) == (0, r, 0, 1)
    tc.set_async(async_)
    tc.set_graphs(graphs)
    pinned = torch.from_numpy(s.view(np.int32)).pin_memory()
    dev = torch.from_numpy(s.view(np.int32)).cuda()
    Sbuf = torch.zeros(64, dtype=torch.int64).pin_memory()
    ref = []
    o = oracle_run(s[:0], r, 11, w)
    for i, k in enumerate(range(0, len(s), w)):
        src = (s, pinned, dev)[i % 3]
        tc.push_batch(src[k:k + w])
        tc.closed_sum_async(Sbuf, i)
        assert o.push_batch(s[k:k + w]) == 0
        ref.append(o.closed_sum())
    assert tc.sync() == 0
    assert Sbuf[: len(ref)].tolist() == ref
    assert_states_equal(tc.state(), o.state(), f"rank handle async={async_} graphs={graphs}")
    assert tc.closed_sum() == o.closed_sum() and tc.estimate() == o.estimate()
    plain = TriangleCounter(r, 11)
    for k in range(0, len(s), w):
        plain.push_batch(s[k:k + w])
    for groups in (1, 7, 100):
        assert tc.group_sums(groups).tolist() == plain.group_sums(groups).tolist()
        assert tc.estimate_mom(groups) == plain.estimate_mom(groups)


@pytest.mark.parametrize("graphs", [False, True])
def test_rank_handle_world1_pair_filter(graphs):
    """The large-batch path (pair filter filled by k_count, evict-first probes, half-full edge-pair table) through
    a rank handle: batches broadcast on the comm stream into alternating receive buffers while the filters
    alternate by batch parity."""
    from paper_1308_2166_b200 import TriangleCounter, nccl_unique_id
    s = rmat(14, 16, 9)
    r, w = 4000, 20000
    tc = TriangleCounter.rank(r, 3, 0, 1, nccl_unique_id(), device=0, w_max_hint=w)
    tc.tune(pair_filter=2, small_batch=1)
    tc.set_graphs(graphs)
    for k in range(0, len(s), w):
        tc.push_batch(s[k:k + w])
    o = oracle_run(s, r, 3, w)
    assert_states_equal(tc.state(), o.state(), f"rank handle + pair filter, graphs={graphs}")
    assert tc.closed_sum() == o.closed_sum()


def test_rank_handle_rejects_bad_batch_and_large_w():
    from paper_1308_2166_b200 import TriangleCounter, nccl_unique_id
    from paper_1308_2166_b200._lib import TC_EDUP, TC_EINVAL
    s = rmat(11, 16, 2)
    tc = TriangleCounter.rank(900, 3, 0, 1, nccl_unique_id(), device=0)
    tc.push_batch(s[:1000])
    before = tc.state()
    bad = np.ascontiguousarray(np.concatenate([s[1000:1100], s[1010:1011, ::-1]]))
    assert tc.push_batch(bad, check=False) == TC_EDUP
    assert_states_equal(tc.state(), before, "rejected")
    assert tc.push_batch(None, check=False, w=10) == TC_EINVAL  # rank 0 must pass the edges
    tc.push_batch(s[1000:9000])  # grows the index (and the broadcast buffers)
    o = oracle_run(s[:1000], 900, 3, 1000)
    assert o.push_batch(s[1000:9000]) == 0
    assert_states_equal(tc.state(), o.state(), "after growth")


def test_rank_counter_world1_bootstrap():
    """dist.RankCounter: the torch-free world-1 bootstrap path of the production multi-GPU driver."""
    from paper_1308_2166_b200.dist import RankCounter
    s = rmat(12, 16, 9)
    rc = RankCounter(2000, 5, 4096)
    dev = torch.from_numpy(s.view(np.int32)).cuda()
    for k in range(0, len(s), 4096):
        rc.push_batch(dev[k:k + 4096])
    o = oracle_run(s, 2000, 5, 4096)
    assert rc.closed_sum() == o.closed_sum() and rc.estimate() == o.estimate()
    assert_states_equal(rc.engine.state(), o.state(), "RankCounter")


def test_multi_single_device_is_plain_handle():
    """tc_create_ex with one device: a plain handle configured by tc_config (strict / graphs / hint)."""
    from paper_1308_2166_b200 import TriangleCounter
    s = rmat(12, 16, 6)
    tc = TriangleCounter.multi(1500, 8, [0], strict=False, graphs=True, w_max_hint=3000)
    for k in range(0, len(s), 3000):
        tc.push_batch(s[k:k + 3000])
    assert tc.sync() == 0
    assert_states_equal(tc.state(), oracle_run(s, 1500, 8, 3000).state(), "tc_create_ex(1)")
