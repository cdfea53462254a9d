"""Per-step parity of the split estimator pass: with TC_TUNE_SPLIT_KERNELS the GPU runs
Ku1 (Step 1), Ku2 (chi^+), Ku3 (level-2 select, PAPER.md:564-569,
761-767), Ku4 (closing edge) and Kr (aggregate) as separate kernels and keeps each step's
values; they must equal the oracle's per-step trace (oracle/indexed.c, the paper's bulk algorithm) after EVERY
batch, and the states must equal both the oracle's and the fused pass's."""
import numpy as np
import pytest

from gpu_common import assert_states_equal
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


def _run(stream, r, seed, sizes, knobs=None):
    from oracle.indexed import IndexedOracle
    from paper_1308_2166_b200 import TriangleCounter
    g = TriangleCounter(r, seed)
    g.tune(split_kernels=1, **(knobs or {}))
    fused = TriangleCounter(r, seed)
    if knobs:
        fused.tune(**knobs)
    o = IndexedOracle(r, seed)
    o.set_trace(True)
    k = 0
    for b, w in enumerate(sizes):
        W = stream[k:k + w]
        k += w
        g.push_batch(W)
        fused.push_batch(W)
        assert o.push_batch(W) == 0
        gs, ot = g.steps(), o.trace()
        for f in ("j", "chi_m", "ld", "rd", "d2", "k2"):
            if not np.array_equal(gs[f], ot[f]):
                i = int(np.nonzero(gs[f] != ot[f])[0][0])
                raise AssertionError(f"batch {b}: step value {f} differs at estimator {i}: {gs[f][i]} vs {ot[f][i]}")
        st = g.state()
        assert np.array_equal(st["closed"], ot["closed"]), f"batch {b}: Step 3 flags"
        assert_states_equal(st, o.state(), f"split pass, batch {b}")
        assert_states_equal(st, fused.state(), f"split vs fused, batch {b}")
        assert g.closed_sum() == o.closed_sum()
    return g


@pytest.mark.parametrize("seed", range(3))
def test_steps_C1(seed):
    s = er(1000, 20000, 1)
    _run(s, 4096, seed, [2048] * 9 + [1568])


@pytest.mark.parametrize("lw", [10, 14])
def test_steps_rmat_hubs(lw):
    s = rmat(14, 16, 3)
    w = 1 << lw
    sizes = [w] * (len(s) // w) + ([len(s) % w] if len(s) % w else [])
    _run(s, 9000, 7 + lw, sizes[:12])


def test_steps_with_index_paths():
    """Split pass over every index path (hub peeling, radix-sort buckets, split partition)."""
    s = rmat(13, 16, 5)
    for knobs in (dict(vbucket_cap=1, vbucket_sort_cap=1), dict(vbucket_arcs=1), dict(small_batch=2)):
        _run(s, 3000, 21, [5000, 5000, 1, 7000, 333], knobs)
