"""Brute-force oracle: the paper's *conceptual* per-estimator bulk update.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain, slow, obviously
correct: every step is the per-estimator rule as PAPER.md states it, with W
scanned by brute force (no index, no sort, no hashing).

Notation follows §4: E = edges seen before the batch
(|E| = m_prev), W = <w_0 .. w_{s-1}> the arriving batch (0-based here; the
paper is 1-based), est_i = (f1, f2, f3, chi).  Positions are 0-based global
stream positions: batch edge k has position m_prev + k.

State per estimator: r1=f1 as (lo, hi) with lo < hi,
p1 its position, r2=f2, p2, c=chi, closed = (f3 != empty).
EMPTY edge = (0xFFFFFFFF, 0xFFFFFFFF), EMPTY position = 2^64-1.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from . import rng

EMPTY_V = 0xFFFFFFFF
EMPTY_E = (EMPTY_V, EMPTY_V)
EMPTY_P = (1 << 64) - 1
C_MAX = (1 << 31) - 1

TC_OK = 0
TC_EINVAL = -1
TC_ESELFLOOP = -3
TC_EDUP = -4
TC_EOVERFLOW = -5


class BatchRejected(Exception):
    def __init__(self, code):
        super().__init__(code)
        self.code = code


@dataclass
class Est:
    r1: tuple = EMPTY_E
    p1: int = EMPTY_P
    r2: tuple = EMPTY_E
    p2: int = EMPTY_P
    c: int = 0
    closed: bool = False


def normalize(u, v):
    """An edge is a size-2 set; store it as (min, max)."""
    u, v = int(u), int(v)
    return (u, v) if u < v else (v, u)


def validate_batch(W):
    """Input contract: reserved id, self-loop, in-batch duplicate.

    The paper assumes a simple graph whose edges arrive exactly once
    (PAPER.md:218-220); a batch that violates it is rejected whole, with
    priority EINVAL > ESELFLOOP > EDUP when several violations occur.
    """
    errs = set()
    seen = set()
    for (u, v) in W:
        u, v = int(u), int(v)
        if u == EMPTY_V or v == EMPTY_V:
            errs.add(TC_EINVAL)
        if u == v:
            errs.add(TC_ESELFLOOP)
        e = normalize(u, v)
        if e in seen:
            errs.add(TC_EDUP)
        seen.add(e)
    for code in (TC_EINVAL, TC_ESELFLOOP, TC_EDUP):
        if code in errs:
            return code
    return TC_OK


def step1_level1(est: Est, E_W, m_prev: int, uniform):
    """Step 1 (§4.2).

    "with probability |W|/(|W|+|E|), replace f1 with an edge uniformly chosen
    from W; otherwise, retain the current edge" -- realised as one draw
    d1 = randInt(|W|+|E|): replace iff d1 >= |E|, with the
    replacement W[d1 - |E|] (reading R2).  A replaced estimator gets
    chi = 0 and, by NBSI clauses 3-4,
    an empty f2/f3 (reading R3).
    """
    s = len(E_W)
    d1 = uniform(1, m_prev + s)
    if d1 >= m_prev:
        j = d1 - m_prev
        est.r1 = E_W[j]
        est.p1 = d1
        est.c = 0
        est.r2 = EMPTY_E
        est.p2 = EMPTY_P
        est.closed = False


def substream_L_R(est: Est, E_lo, E_hi, m_prev: int):
    """Gamma_W(f1) = L u R (Observation), by brute force.

    L = batch edges incident on u that arrive after f1, in rank order
    (rank 0 = the latest, PAPER.md:589-600 and observation 2 at 733-734),
    i.e. in decreasing position; R likewise for v.  u = min endpoint
    (reading R1, which reproduces Fig. 5).
    """
    u, v = est.r1
    k = np.arange(len(E_lo), dtype=np.int64)
    after = (m_prev + k) > est.p1 if est.p1 != EMPTY_P else np.ones(len(E_lo), bool)
    L = k[((E_lo == u) | (E_hi == u)) & after][::-1]
    R = k[((E_lo == v) | (E_hi == v)) & after][::-1]
    return L, R


def step2_level2(est: Est, E_W, E_lo, E_hi, m_prev: int, uniform):
    """Step 2 (§4.3), naming scheme PAPER.md:761-767.

    chi^- = chi, chi^+ = |Gamma_W(f1)|; "with probability chi^-/(chi^-+chi^+)
    keep the current f2; otherwise pick a random edge from Gamma_W(f1).  Then
    update chi to chi^- + chi^+."  Realised as one draw d2 over chi^-+chi^+:
    keep iff d2 < chi^-, else phi = d2 - chi^- names the edge (reading R4); no
    draw when chi^+ = 0.
    """
    L, R = substream_L_R(est, E_lo, E_hi, m_prev)
    chi_m = est.c
    chi_p = len(L) + len(R)
    if chi_p > 0:
        d2 = uniform(2, chi_m + chi_p)
        if d2 >= chi_m:
            phi = d2 - chi_m
            k = int(L[phi]) if phi < len(L) else int(R[phi - len(L)])
            est.r2 = E_W[k]
            est.p2 = m_prev + k
            est.closed = False  # reading R5: a new f2 has no closing edge yet
        est.c = chi_m + chi_p


def closing_pair(r1, r2):
    """The edge that completes the wedge (f1, f2) (NBSI clause 4)."""
    a = set(r1) - set(r2)
    z = set(r2) - set(r1)
    assert len(a) == 1 and len(z) == 1, (r1, r2)
    return normalize(a.pop(), z.pop())


def step3_closing(est: Est, E_W, m_prev: int):
    """Step 3 (§4.4): is the closing edge in W, after f2?

    Reading R6: an already-closed estimator stays closed (edges arrive once,
    PAPER.md:219-220, so its closing edge cannot reappear); for an old f2 every
    batch edge is later, for a fresh f2 the closing edge must have a larger
    position.
    """
    if est.r2 == EMPTY_E or est.closed:
        return
    want = closing_pair(est.r1, est.r2)
    for k, e in enumerate(E_W):
        if e == want and m_prev + k > est.p2:
            est.closed = True
            return


@dataclass
class BruteOracle:
    """r estimators with global ids [first, first+count), Philox-driven (rng.PhiloxDraws)."""

    r: int
    seed: int
    first: int = 0
    count: int | None = None
    m: int = 0
    b: int = 0
    ests: list = field(default_factory=list)

    def __post_init__(self):
        if self.r <= 0:
            raise ValueError("r must be >= 1")
        if self.count is None:
            self.count = self.r - self.first
        self.ests = [Est() for _ in range(self.count)]

    def push_batch(self, W, uniform_factory=None):
        """bulkUpdateAll: Steps 1, 2, 3 for every estimator; all-or-nothing."""
        W = [tuple(map(int, e)) for e in W]
        if len(W) == 0:
            return TC_OK
        code = validate_batch(W)
        if code != TC_OK:
            return code
        E_W = [normalize(u, v) for (u, v) in W]
        E_lo = np.array([e[0] for e in E_W], dtype=np.int64)
        E_hi = np.array([e[1] for e in E_W], dtype=np.int64)
        m_prev = self.m
        ids = np.arange(self.first, self.first + self.count, dtype=np.uint64)
        if uniform_factory is None:
            xlo, xhi = rng.batch_words(self.seed, ids, self.b)
            hooks = [rng.PhiloxDraws(self.seed, int(i), self.b, (int(a), int(c)))
                     for i, a, c in zip(ids, xlo, xhi)]
        else:
            hooks = [uniform_factory(int(i), self.b) for i in ids]
        new = [replace(e) for e in self.ests]  # all-or-nothing: commit only if no estimator overflows
        for est, uniform in zip(new, hooks):
            step1_level1(est, E_W, m_prev, uniform)
            step2_level2(est, E_W, E_lo, E_hi, m_prev, uniform)
            step3_closing(est, E_W, m_prev)
        # overflow guard (reading R13): chi = chi^- + chi^+ is computed exactly; a batch after which some
        # estimator's chi exceeds 2^31 - 1 (bit 31 of the packed word is the closed flag) is rejected whole.
        # Positions and m are unbounded (u64 in the state), so no other limit applies.
        if any(e.c > C_MAX for e in new):
            return TC_EOVERFLOW
        self.ests = new
        self.m += len(W)
        self.b += 1
        return TC_OK

    def state(self):
        n = len(self.ests)
        r1 = np.array([e.r1 for e in self.ests], dtype=np.uint32).reshape(n, 2)
        r2 = np.array([e.r2 for e in self.ests], dtype=np.uint32).reshape(n, 2)
        p1 = np.array([e.p1 for e in self.ests], dtype=np.uint64)
        p2 = np.array([e.p2 for e in self.ests], dtype=np.uint64)
        c = np.array([e.c for e in self.ests], dtype=np.uint32)
        closed = np.array([e.closed for e in self.ests], dtype=np.uint8)
        return dict(r1=r1, p1=p1, r2=r2, p2=p2, c=c, closed=closed)

    def closed_sum(self):
        """S = sum of chi over estimators whose f3 != empty (exact integer)."""
        return sum(e.c for e in self.ests if e.closed)

    def estimate(self):
        """Mean of the coarse estimates X_i = chi_i*|E| if f3 != empty else 0 (Lemma unbiased-est,
        PAPER.md:336-343), evaluated as (double)m * (double)S / (double)r (reading R9)."""
        return float(self.m) * float(self.closed_sum()) / float(self.r)


def coarse_estimates(state, m):
    """X_i per estimator, as exact Python ints."""
    return [int(c) * m if cl else 0 for c, cl in zip(state["c"], state["closed"])]


def median_of_means(state, m, groups):
    """Median-of-means (the paper's aggregate, 887-888) of the coarse estimates
    X_i = c_i*m (closed) else 0.  Reading R9: contiguous groups g = [floor(g*n/G), floor((g+1)*n/G)),
    group mean = (double)m * (double)S_g / (double)|g| with S_g the exact sum of c over the group's
    closed estimators, and the lower median of the G means."""
    c = [int(x) for x in state["c"]]
    cl = [int(x) for x in state["closed"]]
    n = len(c)
    if not (1 <= groups <= n):
        raise ValueError("groups must be in [1, n]")
    means = []
    for g in range(groups):
        lo, hi = g * n // groups, (g + 1) * n // groups
        S_g = sum(c[i] for i in range(lo, hi) if cl[i])
        means.append(float(m) * float(S_g) / float(hi - lo))
    means.sort()
    return means[(groups - 1) // 2]


def required_estimators(eps, delta, m, Delta, tau):
    """r >= 96/eps^2 * m*Delta/tau * log(1/delta) (Theorem mdelta-suffices);
    natural log (reading R10)."""
    import math
    return math.ceil(96.0 / (eps * eps) * (m * Delta / tau) * math.log(1.0 / delta))
