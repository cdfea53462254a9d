"""The exact triangle counter: the ground truth of the accuracy study.

CPU (-m "not gpu"): the two oracle routes -- oracle.exact.triangles (adjacency-set enumeration) and
oracle.exact.triangle_count (tau = sum((A @ A) * A) / 6) -- pinned to closed forms (K_n: C(n, 3);
K_{a,b}: 0; wheel W_n: n; friendship graph F_k: k) and to an O(n^3) brute force on tiny graphs.
GPU (-m gpu): tc_exact_triangles equals the oracle on the same seeded graphs (bit-exact integer), is
invariant under relabelling / reordering / reorientation at sizes the oracle cannot reach, and rejects bad
input with the documented codes (include/tc.h).
"""
import itertools
import math
import random

import numpy as np
import pytest

from oracle import exact
from synth import er, rmat


def complete(n):
    return [(a, b) for a in range(n) for b in range(a + 1, n)]


def bipartite(a, b):
    return [(i, a + j) for i in range(a) for j in range(b)]


def wheel(n):  # hub 0 + cycle 1..n
    return [(0, i) for i in range(1, n + 1)] + [(i, i % n + 1) for i in range(1, n + 1)]


def friendship(k):  # k triangles sharing vertex 0
    return [e for t in range(k) for e in ((0, 2 * t + 1), (0, 2 * t + 2), (2 * t + 1, 2 * t + 2))]


CLOSED = [(complete(2), 0), (complete(3), 1), (complete(12), math.comb(12, 3)), (bipartite(5, 7), 0),
          (wheel(4), 4), (wheel(9), 9), (friendship(6), 6), ([], 0)]


def brute(stream):
    E = {tuple(sorted(e)) for e in stream}
    V = sorted({x for e in E for x in e})
    return sum(1 for a, b, c in itertools.combinations(V, 3) if (a, b) in E and (a, c) in E and (b, c) in E)


@pytest.mark.parametrize("i", range(len(CLOSED)))
def test_oracle_closed_forms(i):
    g, tau = CLOSED[i]
    assert len(exact.triangles(g)) == tau
    assert exact.triangle_count(g) == tau


@pytest.mark.parametrize("seed", range(6))
def test_oracle_brute_tiny(seed):
    rnd = random.Random(seed)
    n = rnd.randint(5, 14)
    pairs = complete(n)
    rnd.shuffle(pairs)
    g = [tuple(rnd.sample(p, 2)) for p in pairs[:rnd.randint(0, len(pairs))]]
    t = brute(g)
    assert len(exact.triangles(g)) == t
    assert exact.triangle_count(g) == t


def test_oracle_routes_agree_C1():
    g = er(1000, 20000, 4)
    assert len(exact.triangles(g)) == exact.triangle_count(g)


# ------------------------------------------------------------------------------------------------ GPU


def _relabel(g, seed):
    rng = np.random.default_rng(seed)
    g = np.asarray(g, dtype=np.uint32).reshape(-1, 2)
    ids = np.unique(g)
    new = rng.choice(np.uint64(0xFFFFFFFE), size=len(ids), replace=False).astype(np.uint32)
    lut = dict(zip(ids.tolist(), new.tolist()))
    h = np.vectorize(lut.get, otypes=[np.uint32])(g) if len(g) else g
    h = h[rng.permutation(len(h))]
    flip = rng.random(len(h)) < 0.5
    h[flip] = h[flip][:, ::-1]
    return np.ascontiguousarray(h)


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(len(CLOSED)))
def test_gpu_closed_forms(i):
    from paper_1308_2166_b200 import exact_triangles
    g, tau = CLOSED[i]
    assert exact_triangles(np.asarray(g, dtype=np.uint32).reshape(-1, 2)) == tau
    if len(g):
        assert exact_triangles(_relabel(g, i)) == tau


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(4))
def test_gpu_equals_oracle_random(seed):
    from paper_1308_2166_b200 import exact_triangles
    rnd = random.Random(100 + seed)
    n = rnd.randint(20, 300)
    g = er(n, rnd.randint(1, min(4000, n * (n - 1) // 2)), seed)
    assert exact_triangles(g) == exact.triangle_count(g)


@pytest.mark.gpu
def test_gpu_equals_oracle_C1_and_rmat():
    import torch
    from paper_1308_2166_b200 import exact_triangles
    g = er(1000, 20000, 4)  # configs[0]
    tau = exact.triangle_count(g)
    assert exact_triangles(g) == tau
    dev = torch.from_numpy(g.view(np.int32)).cuda()  # device input
    assert exact_triangles(dev) == tau
    h = rmat(12, 16, 7)  # power-law hubs: the warp-per-arc path runs
    assert exact_triangles(h) == exact.triangle_count(h)


@pytest.mark.gpu
def test_gpu_invariances_large():
    """R-MAT scale 18 (~4M edges, beyond the oracle): relabelling, reordering and reorientation leave tau
    unchanged; a disjoint union adds."""
    from paper_1308_2166_b200 import exact_triangles
    g = rmat(18, 16, 3)
    t = exact_triangles(g)
    assert t > 0
    assert exact_triangles(_relabel(g, 5)) == t
    k = complete(40)
    off = int(g.max()) + 1
    u = np.concatenate([g, np.asarray(k, dtype=np.uint32) + off])
    assert exact_triangles(u) == t + math.comb(40, 3)


@pytest.mark.gpu
def test_gpu_errors():
    from paper_1308_2166_b200 import TCError, exact_triangles
    from paper_1308_2166_b200._lib import TC_EDUP, TC_EINVAL, TC_ESELFLOOP
    cases = [([(1, 2), (3, 3)], TC_ESELFLOOP), ([(1, 2), (2, 1)], TC_EDUP), ([(1, 2), (1, 2), (2, 3)], TC_EDUP),
             ([(0xFFFFFFFF, 2)], TC_EINVAL)]
    for g, code in cases:
        with pytest.raises(TCError) as ei:
            exact_triangles(np.asarray(g, dtype=np.uint32))
        assert ei.value.code == code
    assert exact_triangles(np.zeros((0, 2), dtype=np.uint32)) == 0
