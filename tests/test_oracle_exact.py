"""Closed-form and brute-force pins of the whole estimator (oracle vs mathematics).

* E[X] = tau (Lemma unbiased-est) exactly, by rational enumeration.
* E[X^2] = m * sum_t C(t): from Claim discovery-prob X = m*C(t) w.p.
  1/(m*C(t)) per triangle, 0 otherwise.
* The final state distribution does not depend on the batching; batch size 1 is
  "the familiar reservoir sampling": P(f1 = e) = 1/m exactly.
* NBSI clauses hold for every estimator after every batch:
  c == |Gamma_S(r1)|, r2 in Gamma_S(r1), closed <=> closing edge after r2.
* brute-force oracle == bulk (indexed) oracle, bit for bit.
"""
import random
from fractions import Fraction

import numpy as np
import pytest

from oracle import exact, indexed, nbsi
from synth import er


def _tiny(seed, n=6, m=9):
    rnd = random.Random(seed)
    pairs = [(a, b) for a in range(n) for b in range(a + 1, n)]
    rnd.shuffle(pairs)
    return [tuple(rnd.sample(p, 2)) for p in pairs[:m]]


def _batchings(m):
    return [[1] * m, [2] * (m // 2) + [m % 2] * (m % 2), [3] * (m // 3) + ([m % 3] if m % 3 else []), [m]]


@pytest.mark.parametrize("seed", range(6))
def test_exact_moments_and_batch_invariance(seed):
    s = _tiny(seed, n=6, m=8 + seed % 3)
    tau, sumC, m = exact.moments(s)
    dists = []
    for bs in _batchings(m):
        bs = [b for b in bs if b]
        d = exact.enumerate_distribution(s, bs)
        assert sum(d.values()) == 1
        ex, ex2 = exact.dist_moments(d, m)
        assert ex == tau, (bs, ex, tau)
        assert ex2 == m * sumC, (bs, ex2, m * sumC)
        dists.append(d)
    for d in dists[1:]:
        assert d == dists[0]
    # Claim discovery-prob: P({f1,f2,f3} = t) = 1/(m C(t)) for every triangle t
    pos = {nbsi.normalize(*e): i for i, e in enumerate(s)}
    g = exact.gamma_sizes(s)
    for t in exact.triangles(s):
        e1, e2, e3 = sorted(t, key=lambda e: pos[e])
        p = sum(pr for st, pr in dists[0].items() if st[5] and st[0] == e1 and st[2] == e2)
        assert p == Fraction(1, m * g[pos[e1]])


def test_reservoir_marginal_uniform():
    s = _tiny(11, n=7, m=12)
    m = len(s)
    for bs in ([1] * m, [5, 7], [m]):
        d = exact.enumerate_distribution(s, bs)
        marg = {}
        for st, pr in d.items():
            marg[st[0]] = marg.get(st[0], 0) + pr
            assert s[st[1]] and nbsi.normalize(*s[st[1]]) == st[0]  # p1 is r1's position
        assert len(marg) == m and all(v == Fraction(1, m) for v in marg.values())


def test_gamma_helpers_brute():
    s = _tiny(3, n=8, m=20)
    g = exact.gamma_sizes(s)
    assert g == [exact.gamma_brute(s, i) for i in range(len(s))]


def _check_nbsi(stream_prefix, st):
    """NBSI clauses 2-4 for every estimator, by brute force on the prefix."""
    E = [nbsi.normalize(*e) for e in stream_prefix]
    m = len(E)
    for i in range(st["c"].shape[0]):
        r1 = tuple(int(x) for x in st["r1"][i])
        p1 = int(st["p1"][i])
        assert 0 <= p1 < m and E[p1] == r1
        gam = [j for j in range(p1 + 1, m) if len(set(E[j]) & set(r1)) == 1]
        assert int(st["c"][i]) == len(gam)
        r2 = tuple(int(x) for x in st["r2"][i])
        if not gam:
            assert r2 == nbsi.EMPTY_E and int(st["p2"][i]) == nbsi.EMPTY_P and st["closed"][i] == 0
            continue
        p2 = int(st["p2"][i])
        assert p2 in gam and E[p2] == r2
        want = nbsi.closing_pair(r1, r2)
        closing = any(E[j] == want for j in range(p2 + 1, m))
        assert bool(st["closed"][i]) == closing


@pytest.mark.parametrize("seed", range(4))
def test_invariants_and_brute_eq_bulk(seed):
    s = er(40, 300, seed + 100)
    r = 300
    bo = nbsi.BruteOracle(r, seed)
    io = indexed.IndexedOracle(r, seed)
    rnd = random.Random(seed)
    k = 0
    while k < len(s):
        w = rnd.choice([1, 2, 7, 33, 64, 150])
        W = s[k:k + w]
        assert bo.push_batch(W) == 0 and io.push_batch(W) == 0
        k += len(W)
        a, b = bo.state(), io.state()
        for f in a:
            np.testing.assert_array_equal(a[f], b[f], err_msg=f)
        _check_nbsi(s[:k], a)
    assert bo.closed_sum() == io.closed_sum()
    assert bo.estimate() == io.estimate()
    assert io.counters()[0] == len(s)


def test_brute_eq_bulk_C1():
    """C1 (BASELINE.json configs[0]) end to end: brute force == bulk oracle on every field."""
    s = er(1000, 20000, 1)
    bo = nbsi.BruteOracle(4096, 42)
    io = indexed.IndexedOracle(4096, 42)
    for k in range(0, len(s), 2048):
        assert bo.push_batch(s[k:k + 2048]) == 0 and io.push_batch(s[k:k + 2048]) == 0
    a, b = bo.state(), io.state()
    for f in a:
        np.testing.assert_array_equal(a[f], b[f], err_msg=f)
    assert bo.closed_sum() == io.closed_sum() > 0


def test_sharded_oracle_equals_whole():
    """Estimator sharding by global id: shards [first, first+count) reproduce the unsharded states
    (the RNG is keyed by global id, reading R7)."""
    s = er(60, 500, 9)
    whole = indexed.IndexedOracle(1000, 5)
    parts = [indexed.IndexedOracle(1000, 5, f, c) for f, c in ((0, 300), (300, 1), (301, 699))]
    for k in range(0, len(s), 64):
        assert whole.push_batch(s[k:k + 64]) == 0
        for p in parts:
            assert p.push_batch(s[k:k + 64]) == 0
    a = whole.state()
    for f in a:
        np.testing.assert_array_equal(a[f], np.concatenate([p.state()[f] for p in parts]))
    assert whole.closed_sum() == sum(p.closed_sum() for p in parts)


@pytest.mark.parametrize("kind", ["brute", "bulk"])
def test_error_paths_all_or_nothing(kind):
    mk = (lambda: nbsi.BruteOracle(50, 3)) if kind == "brute" else (lambda: indexed.IndexedOracle(50, 3))
    o = mk()
    s = er(20, 60, 2)
    assert o.push_batch(s[:30]) == 0
    before = o.state()
    assert o.push_batch([]) == 0  # w = 0: no-op
    bad = [
        (list(map(tuple, s[30:40])) + [(5, 5)], nbsi.TC_ESELFLOOP),
        (list(map(tuple, s[30:40])) + [tuple(s[31][::-1])], nbsi.TC_EDUP),
        ([(1, 0xFFFFFFFF)] + list(map(tuple, s[30:40])), nbsi.TC_EINVAL),
        ([(4, 4), (0xFFFFFFFF, 2), (1, 2), (2, 1)], nbsi.TC_EINVAL),  # priority EINVAL > ESELFLOOP > EDUP
        ([(4, 4), (1, 2), (2, 1)], nbsi.TC_ESELFLOOP),
    ]
    for W, code in bad:
        assert o.push_batch(W) == code
        after = o.state()
        for f in before:
            np.testing.assert_array_equal(before[f], after[f])
    assert o.push_batch(s[30:]) == 0
    # the rejected batches did not advance the batch index: same as a clean run
    clean = mk()
    clean.push_batch(s[:30])
    clean.push_batch(s[30:])
    for f in before:
        np.testing.assert_array_equal(o.state()[f], clean.state()[f])


def test_mom_and_sizing():
    # closed estimators with c = (5, 1, 9, 3, 7, 2), m = 1 -> X = c
    st = dict(c=np.array([5, 1, 9, 3, 7, 2]), closed=np.ones(6, np.uint8))
    assert nbsi.median_of_means(st, 1, 1) == 27 / 6
    assert nbsi.median_of_means(st, 1, 6) == 3  # lower median of the values
    assert nbsi.median_of_means(st, 1, 3) == 4.5  # group means 3, 6, 4.5 -> median 4.5
    assert nbsi.median_of_means(st, 1, 2) == 4.0  # group means 5, 4 -> lower median 4
    st2 = dict(c=np.array([5, 1, 9, 3]), closed=np.array([1, 0, 0, 1], np.uint8))
    assert nbsi.median_of_means(st2, 10, 2) == 15.0  # group means 50/2, 30/2 -> lower median 15
    # Theorem mdelta-suffices: 96/eps^2 * m*Delta/tau * ln(1/delta)
    import math
    assert nbsi.required_estimators(0.5, math.exp(-1), 10, 4, 20) == math.ceil(96 / 0.25 * 2.0)
