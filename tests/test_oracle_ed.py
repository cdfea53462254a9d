"""Pins of the event-driven oracle (oracle/ed.py; reading R17).

* Skip-sampler law: P(next_after(t) > s) = t/s (the product of the per-edge coins 1 - 1/q, q = t+1 .. s),
  checked against that closed form on 2*10^4 Philox-driven samples per t, and exactly on its building blocks
  (epoch law, proposal range, acceptance probabilities) by enumerating the sampler's integer branches.
* The whole estimator under the ideal skip laws, by exact rational enumeration: its joint outcome distribution
  over (f1, p1, f2, p2, chi, closed) EQUALS the bulk oracle's at batch size 1 (exact.enumerate_distribution, the
  paper's coin-per-edge reservoir) -- hence E[X] = tau and E[X^2] = m * sum C(t)
  (Lemma unbiased-est, Claim discovery-prob), also asserted directly.
* NBSI clauses by brute force for every estimator after every batch of Philox runs, plus
  J > m and K > chi (a pending event lies in the future).
* Batch invariance: the state after a prefix does not depend on the batching.
* Unbiasedness over seeds (statistical).
"""
import random
from fractions import Fraction

import numpy as np
import pytest

from oracle import ed, exact, nbsi
from synth import er

from test_oracle_exact import _check_nbsi, _tiny


class _Words:
    """A scripted word stream (for branch-by-branch checks of the sampler)."""

    def __init__(self, words):
        self.words, self.ev = list(words), 0

    def next(self):
        w = self.words[self.ev]
        self.ev += 1
        return w


@pytest.mark.parametrize("t", [1, 2, 5, 1000, 1 << 20])
def test_next_after_tail_law(t):
    n = 20000
    vals = np.array([ed.next_after(t, ed.WordStream(7, i)) for i in range(n)], dtype=np.float64)
    assert (vals > t).all()
    for f in (1.5, 2, 3, 4, 16, 100):
        s = int(t * f)
        p = t / s
        emp = float((vals > s).mean())
        sd = (p * (1 - p) / n) ** 0.5
        assert abs(emp - p) <= 5 * sd + 1e-12, (t, s, emp, p)


def test_next_after_small_t_pmf():
    """t = 1: P(T = s) = 1/(s(s-1)) for s = 2..9, chi-square over 4*10^4 draws."""
    n = 40000
    vals = [ed.next_after(1, ed.WordStream(3, i)) for i in range(n)]
    obs = np.bincount(np.minimum(vals, 10), minlength=11)[2:11]
    exp = np.array([n / (s * (s - 1)) for s in range(2, 10)] + [n / 9])
    chi2 = float(((obs - exp) ** 2 / exp).sum())
    assert chi2 < 30.0, (chi2, obs, exp)  # 8 dof: P(chi2 > 30) < 3e-4


def test_next_after_branches():
    """The sampler's integer branches, driven by chosen words."""
    assert ed.next_after(0, _Words([])) == 1
    assert ed.next_after(5, _Words([0])) == ed.INF                       # x = 0: epoch >= 64
    assert ed.next_after(1 << 20, _Words([1 << 11])) == ed.INF          # L = 2^31 > HMAX
    # epoch k = 1 for t = 3 (L = 6): proposal U = hi64(x * 6); s = 7 + U; accept U[0,s-1) < 6 and U[0,s) < 7
    x_u = (2 << 64) // 6 + 2          # U = 2 -> s = 9 (low word >= n: no rejection test)
    x_a = 0                            # U[0, 8) = 0 < 6
    x_b = (5 << 64) // 9 + 2           # U[0, 9) = 5 < 7
    assert ed.next_after(3, _Words([0b10, x_u, x_a, x_b])) == 9
    # the same with the first acceptance failing (U[0, 8) = 7 >= 6): the next proposal is taken
    x_rej = (1 << 64) - 1
    assert ed.next_after(3, _Words([0b10, x_u, x_rej, x_u, x_a, x_b])) == 9


def test_acceptance_probabilities_exact():
    """Inside an epoch, proposal uniform over (L, 2L] and acceptance L/(s-1) * (L+1)/s give
    P(T = s | epoch) = 2L/(s(s-1)) exactly; and sum_k P(epoch k) * that = t/(s(s-1))."""
    for t in (1, 3, 7):
        for k in range(0, 4):
            L = t << k
            acc = {s: Fraction(L, s - 1) * Fraction(L + 1, s) for s in range(L + 1, 2 * L + 1)}
            assert all(0 < a <= 1 for a in acc.values())
            tot = sum(acc.values())
            for s, a in acc.items():
                assert a / tot == Fraction(2 * L, s * (s - 1))
                assert Fraction(1, 2 ** (k + 1)) * a / tot == ed.next_after_law(t, s)


@pytest.mark.parametrize("seed", range(6))
def test_exact_distribution_equals_bulk_reservoir(seed):
    s = _tiny(seed, n=6, m=7 + seed % 3)
    m = len(s)
    d_ed = ed.enumerate_outcomes(s)
    assert sum(d_ed.values()) == 1
    conv = {}
    for (f1, t1, f2, t2, chi, closed), p in d_ed.items():
        key = (f1, t1 - 1 if t1 else nbsi.EMPTY_P, f2, t2 - 1 if t2 else nbsi.EMPTY_P, chi, closed)
        conv[key] = conv.get(key, Fraction(0)) + p
    d_bulk = exact.enumerate_distribution(s, [1] * m)
    assert conv == d_bulk
    tau, sumC, _ = exact.moments(s)
    ex, ex2 = exact.dist_moments(conv, m)
    assert ex == tau and ex2 == m * sumC


def test_exact_distribution_fig2_like_triangle_rich():
    """K4 plus a pendant path (4 triangles): E[X] = tau, E[X^2] = m sum C."""
    s = [(1, 2), (1, 3), (2, 3), (3, 4), (1, 4), (2, 4), (4, 5)]
    d = ed.enumerate_outcomes(s)
    ex = sum(p * (k[4] * len(s) if k[5] else 0) for k, p in d.items())
    ex2 = sum(p * (k[4] * len(s) if k[5] else 0) ** 2 for k, p in d.items())
    tau, sumC, m = exact.moments(s)
    assert tau == 4 and ex == tau and ex2 == m * sumC


def _check_events(st, m):
    for i in range(len(st["c"])):
        assert int(st["J"][i]) > m
        if int(st["p1"][i]) != nbsi.EMPTY_P:
            assert int(st["K"][i]) > int(st["c"][i])


@pytest.mark.parametrize("seed", range(3))
def test_nbsi_after_every_batch_and_batch_invariance(seed):
    s = er(30, 160, seed + 40)
    r = 60
    rnd = random.Random(seed)
    a = ed.EventOracle(r, seed)
    b = ed.EventOracle(r, seed)
    k = 0
    while k < len(s):
        w = rnd.choice([1, 3, 17, 40])
        assert a.push_batch(s[k:k + w]) == 0
        k = min(k + w, len(s))
        st = a.state()
        _check_nbsi(s[:k], st)
        _check_events(st, k)
    assert b.push_batch(s) == 0  # one batch
    sa, sb = a.state(), b.state()
    for f in sa:
        np.testing.assert_array_equal(sa[f], sb[f], err_msg=f)
    assert a.closed_sum() == b.closed_sum()


def test_rejections_all_or_nothing():
    o = ed.EventOracle(20, 1)
    assert o.push_batch([(1, 2), (2, 3)]) == 0
    before = o.state()
    assert o.push_batch([(3, 4), (4, 3)]) == nbsi.TC_EDUP
    assert o.push_batch([(5, 5)]) == nbsi.TC_ESELFLOOP
    after = o.state()
    for f in before:
        np.testing.assert_array_equal(before[f], after[f])
    assert o.m == 2


def test_unbiased_over_seeds():
    s = er(25, 120, 5)
    tau = exact.triangle_count(s)
    assert tau > 0
    ests = []
    for seed in range(30):
        o = ed.EventOracle(200, seed)
        assert o.push_batch(s) == 0
        ests.append(o.estimate())
    mean = float(np.mean(ests))
    sd = float(np.std(ests)) / len(ests) ** 0.5
    assert abs(mean - tau) <= 5 * sd + 1e-9, (mean, tau, sd)
