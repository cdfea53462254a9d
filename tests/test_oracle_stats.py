"""Statistical pins of the Philox-driven oracle against the paper's claims.

Bounds come from closed forms (no fitted constants):
* mean over S seeds: |mean - tau| <= 4 sqrt(Var[X] / (r S)), Var[X] = m sum_t C(t) - tau^2
  (E[X] = tau, Lemma unbiased-est; E[X^2] from Claim discovery-prob 348-368);
* sample variance vs Var[X] within 5 sd, the sd from the 4th central moment, using
  E[X^k] = sum_t (m C(t))^(k-1);
* chi-square goodness of fit (p > 1e-4) for: f1 uniform over E (NBSI clause 1), f2 uniform over
  Gamma(f1) (clause 3), and per-triangle discovery frequencies 1/(m C(t)) (Claim discovery-prob).
"""
import math
from collections import Counter

import numpy as np
from scipy import stats

from oracle import exact, indexed, nbsi
from synth import er


def _run(stream, r, seed, w):
    o = indexed.IndexedOracle(r, seed)
    for k in range(0, len(stream), w):
        assert o.push_batch(stream[k:k + w]) == 0
    return o


def test_mean_over_seeds_C1():
    s = er(1000, 20000, 1)
    tau, sumC, m = exact.moments([tuple(e) for e in s])
    var = m * sumC - tau * tau
    r, S = 4096, 60
    ests = [_run(s, r, seed, 2048).estimate() for seed in range(S)]
    mean = sum(ests) / S
    bound = 4.0 * math.sqrt(var / (r * S))
    assert abs(mean - tau) <= bound, (mean, tau, bound)
    # per-run spread is consistent with Var[X]/r (loose: within a factor 1.5 of the closed form)
    sd_run = float(np.std(ests, ddof=1))
    assert 0.6 < sd_run / math.sqrt(var / r) < 1.5


def test_variance_closed_form():
    s = [tuple(e) for e in er(60, 500, 4)]
    Cs = exact.C_values(s)
    m, tau = len(s), len(Cs)
    EX = [None, tau, m * sum(Cs), m * m * sum(c * c for c in Cs), m ** 3 * sum(c ** 3 for c in Cs)]
    var = EX[2] - tau ** 2
    mu4 = EX[4] - 4 * tau * EX[3] + 6 * tau ** 2 * EX[2] - 3 * tau ** 4
    N = 200_000
    o = _run(s, N, 77, 37)
    st = o.state()
    X = np.where(st["closed"] == 1, st["c"].astype(np.float64) * m, 0.0)
    assert abs(X.mean() - tau) <= 5 * math.sqrt(var / N)
    sd_s2 = math.sqrt((mu4 - var * var) / N)
    assert abs(X.var(ddof=1) - var) <= 5 * sd_s2, (X.var(ddof=1), var, sd_s2)


def test_level1_and_level2_uniform():
    s = [tuple(e) for e in er(12, 40, 8)]
    m = len(s)
    N = 40_000
    o = _run(s, N, 5, 7)
    st = o.state()
    counts = np.bincount(st["p1"].astype(np.int64), minlength=m)
    assert stats.chisquare(counts).pvalue > 1e-4
    # f2 | f1 uniform over Gamma_S(f1): pool chi-square over f1 values
    g = exact.gamma_sizes(s)
    chi, dof = 0.0, 0
    for p1 in range(m):
        sel = st["p1"] == p1
        if g[p1] < 2 or sel.sum() < 20:
            continue
        c2 = Counter(int(x) for x in st["p2"][sel])
        E = [nbsi.normalize(*e) for e in s]
        r1 = E[p1]
        gam = [j for j in range(p1 + 1, m) if len(set(E[j]) & set(r1)) == 1]
        assert set(c2) <= set(gam)
        obs = np.array([c2.get(j, 0) for j in gam], dtype=float)
        exp = obs.sum() / len(gam)
        chi += float(((obs - exp) ** 2 / exp).sum())
        dof += len(gam) - 1
    assert stats.chi2.sf(chi, dof) > 1e-4


def test_claim1_discovery_frequencies():
    s = [tuple(e) for e in er(9, 22, 3)]
    m = len(s)
    N = 300_000
    o = _run(s, N, 11, 5)
    st = o.state()
    E = [nbsi.normalize(*e) for e in s]
    pos = {e: i for i, e in enumerate(E)}
    g = exact.gamma_sizes(s)
    tris = exact.triangles(s)
    assert len(tris) >= 3
    got = Counter()
    for i in np.nonzero(st["closed"])[0]:
        t = frozenset({tuple(int(x) for x in st["r1"][i]), tuple(int(x) for x in st["r2"][i]),
                       nbsi.closing_pair(tuple(int(x) for x in st["r1"][i]), tuple(int(x) for x in st["r2"][i]))})
        got[t] += 1
    assert set(got) <= set(tris)
    probs = [1.0 / (m * g[min(pos[e] for e in t)]) for t in tris]
    obs = [got.get(t, 0) for t in tris] + [N - sum(got.values())]
    exp = [N * p for p in probs] + [N * (1 - sum(probs))]
    assert stats.chisquare(obs, exp).pvalue > 1e-4
