"""Event-driven oracle: neighborhood sampling with skip-sampled reservoirs.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain and slow: every estimator sees every edge, one at a
time, exactly as the sequential neighborhood-sampling rule of §3.1 maintains NBSI:

    edge e_t arrives (t = 1, 2, ... is its 1-based stream time)
    * with probability 1/t:           f1 <- e_t, chi <- 0, f2 <- empty, f3 <- empty         (clause 1)
    * else if e_t is adjacent to f1:  chi <- chi + 1                                        (clause 2)
                                      with probability 1/chi: f2 <- e_t, f3 <- empty        (clause 3)
                                      else if e_t closes the wedge (f1, f2): f3 <- e_t      (clause 4)

(batch size 1 of bulkUpdateAll is "the familiar reservoir sampling"; the bulk algorithm of
§4 maintains the same invariant per batch).  What makes this mode different from ``nbsi`` is WHICH random bits
decide the two 1/t and 1/chi coins -- DESIGN.md reading R17: each reservoir draws, when it is (re)filled, the
time of its NEXT replacement by skip sampling,

    J  = next_after(t)     when f1 is taken at time t: the next time f1 will be replaced,
    K  = next_after(chi)   when f2 is taken at count chi (K = 1 for a fresh f1): the count at which f2 is next
                           replaced,

with P(next_after(t) > s) = t / s for every s >= t (the product of (1 - 1/q) over q = t+1 .. s), i.e. exactly
the law of the per-edge coins.  Then "t == J" and "chi == K" replace the coins, the outcome law per estimator is
the sequential algorithm's, and, because the draws belong to the estimator's own event sequence, the state after
any prefix of the stream does not depend on how the stream was cut into batches.

The sampler (reading R17, written out step by step; every branch is exact integer arithmetic):

    next_after(0) = 1                                  (the first edge always fills the reservoir)
    t >= 1:  epoch  k = number of trailing zero bits of a 64-bit word (P(k) = 2^-(k+1); x = 0 -> INF)
             L = t * 2^k;  if L > HMAX: return INF       (then T > L > HMAX: never reached, m <= HMAX)
             repeat:  s = L + 1 + U[0, L)                (uniform proposal over the epoch (L, 2L])
                      accept with probability L/(s-1) * (L+1)/s:  U[0, s-1) < L, then U[0, s) < L+1
             return s (INF if s > HMAX)
    Inside epoch k, P(T = s) = t/(s(s-1)) / (t/L - t/(2L)) = 2L/(s(s-1)); the proposal is uniform and the
    acceptance L(L+1)/(s(s-1)) <= 1 is proportional to it, so the accepted s has exactly that law, and
    P(epoch k) = P(L < T <= 2L) = t/L - t/(2L) = 2^-(k+1).

Random words: the estimator's 64-bit word stream n = 0, 1, 2, ...: Philox4x32-10 block
ctr = (id lo, id hi, n >> 1, 0xED5A0000), key = (seed lo, seed hi), word (x | y << 32) for even n,
(z | w << 32) for odd n; U[0, n) is Lemire's multiply-shift with rejection, each retry taking the next word.
``ev`` counts the words an estimator has used.

Overflow (reading R17c): chi <= deg(u) + deg(v); a batch after which some vertex would have degree > 2^30 - 1
is rejected whole (TC_EOVERFLOW), which keeps chi <= 2^31 - 2.
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np

from . import rng
from .nbsi import EMPTY_E, EMPTY_P, TC_EOVERFLOW, TC_OK, normalize, validate_batch

HMAX = (1 << 31) - 1          # largest stream time / count a sampler result is kept for (m < 2^31)
INF = 0xFFFFFFFF              # "never" (beyond HMAX)
DEG_MAX = (1 << 30) - 1       # reading R17c
ED_CTR_W = 0xED5A0000


class WordStream:
    """The 64-bit random words of one estimator (global id ``i``), consumed in order."""

    __slots__ = ("seed", "i", "ev")

    def __init__(self, seed: int, i: int, ev: int = 0):
        self.seed, self.i, self.ev = seed, i, ev

    def next(self) -> int:
        n = self.ev
        self.ev += 1
        blk = rng.philox4x32_10((self.i & rng.MASK32, (self.i >> 32) & rng.MASK32, (n >> 1) & rng.MASK32, ED_CTR_W),
                                (self.seed & rng.MASK32, (self.seed >> 32) & rng.MASK32))
        return rng.words64(blk)[n & 1]


def uniform(n: int, ws) -> int:
    """U[0, n): Lemire's multiply-shift; a rejected word is replaced by the NEXT word of the stream."""
    x = ws.next()
    p = x * n
    if (p & rng.MASK64) < n:
        thresh = ((1 << 64) - n) % n
        while (p & rng.MASK64) < thresh:
            x = ws.next()
            p = x * n
    return p >> 64


def next_after(t: int, ws) -> int:
    """The next replacement time of a size-1 reservoir that was (re)filled at time t (reading R17)."""
    if t == 0:
        return 1
    x = ws.next()
    if x == 0:
        return INF
    k = (x & -x).bit_length() - 1  # trailing zeros
    L = t << k
    if L > HMAX:
        return INF
    while True:
        s = L + 1 + uniform(L, ws)
        if uniform(s - 1, ws) >= L:
            continue
        if uniform(s, ws) >= L + 1:
            continue
        return s if s <= HMAX else INF


def next_after_law(t: int, s: int) -> Fraction:
    """P(next_after(t) = s) = t / (s (s-1)) for s > t >= 1 (the law the sampler must have)."""
    return Fraction(t, s * (s - 1))


def closing_pair(f1, f2):
    """NBSI clause 4: the edge completing the wedge (f1, f2)."""
    a = set(f1) - set(f2)
    z = set(f2) - set(f1)
    return normalize(a.pop(), z.pop())


class EventEst:
    """One estimator: f1, f2 as (lo, hi) with 1-based times t1, t2 (0 = empty), chi, closed, J, K, ev."""

    __slots__ = ("f1", "t1", "f2", "t2", "chi", "closed", "J", "K", "B", "ws")

    def __init__(self, ws):
        self.f1, self.t1, self.f2, self.t2 = EMPTY_E, 0, EMPTY_E, 0
        self.chi, self.closed = 0, False
        self.J = 1  # next_after(0)
        self.K = INF
        self.B = 0
        self.ws = ws

    def see(self, e, t, deg):
        """Edge e (normalised) arrives at time t; ``deg`` = vertex degrees including e (for B only)."""
        if t == self.J:                                   # clause 1: f1 <- e_t
            self.f1, self.t1 = e, t
            self.chi, self.f2, self.t2, self.closed = 0, EMPTY_E, 0, False
            self.B = deg[e[0]] + deg[e[1]]                 # so that chi = deg(u) + deg(v) - B later
            self.J = self.ws.next_after(t)
            self.K = 1                                    # next_after(0): the first neighbour is always taken
        elif self.t1 and (e[0] in self.f1 or e[1] in self.f1):   # clause 2: e in Gamma(f1)
            self.chi += 1
            if self.chi == self.K:                        # clause 3: f2 <- e_t with probability 1/chi
                self.f2, self.t2, self.closed = e, t, False
                self.K = self.ws.next_after(self.chi)
            elif self.t2 and not self.closed and e == closing_pair(self.f1, self.f2):
                self.closed = True                        # clause 4: f3 = e_t > f2


class _Sampler:
    """ws.next_after(t) through the Philox word stream (the production rule)."""

    __slots__ = ("w",)

    def __init__(self, w: WordStream):
        self.w = w

    def next_after(self, t):
        return next_after(t, self.w)

    @property
    def ev(self):
        return self.w.ev


class EventOracle:
    """r estimators with global ids [first, first + count), each fed every edge in stream order."""

    def __init__(self, r: int, seed: int, first: int = 0, count: int | None = None, sampler_factory=None):
        if r <= 0:
            raise ValueError("r must be >= 1")
        self.r, self.seed, self.first = r, seed, first
        self.count = r - first if count is None else count
        make = sampler_factory or (lambda i: _Sampler(WordStream(seed, i)))
        self.ests = [EventEst(make(first + j)) for j in range(self.count)]
        self.m = 0
        self.deg = {}

    def push_batch(self, W) -> int:
        """All-or-nothing: invalid batches (reserved id, self loop, in-batch duplicate) and batches that would
        push a vertex degree past DEG_MAX are rejected before any estimator sees them."""
        W = [tuple(map(int, e)) for e in W]
        if not W:
            return TC_OK
        code = validate_batch(W)
        if code != TC_OK:
            return code
        E = [normalize(u, v) for (u, v) in W]
        add = {}
        for e in E:
            for x in e:
                add[x] = add.get(x, 0) + 1
        if any(self.deg.get(x, 0) + d > DEG_MAX for x, d in add.items()):
            return TC_EOVERFLOW
        for e in E:
            self.m += 1
            for x in e:
                self.deg[x] = self.deg.get(x, 0) + 1
            for est in self.ests:
                est.see(e, self.m, self.deg)
        return TC_OK

    def state(self):
        n = len(self.ests)
        pos = lambda t: EMPTY_P if t == 0 else t - 1  # noqa: E731  (0-based positions, as nbsi)
        return dict(
            r1=np.array([e.f1 for e in self.ests], dtype=np.uint32).reshape(n, 2),
            p1=np.array([pos(e.t1) for e in self.ests], dtype=np.uint64),
            r2=np.array([e.f2 for e in self.ests], dtype=np.uint32).reshape(n, 2),
            p2=np.array([pos(e.t2) for e in self.ests], dtype=np.uint64),
            c=np.array([e.chi for e in self.ests], dtype=np.uint32),
            closed=np.array([e.closed for e in self.ests], dtype=np.uint8),
            J=np.array([e.J for e in self.ests], dtype=np.uint32),
            K=np.array([e.K if e.t1 else INF for e in self.ests], dtype=np.uint32),
            ev=np.array([e.ws.ev for e in self.ests], dtype=np.uint64),
        )

    def closed_sum(self) -> int:
        return sum(e.chi for e in self.ests if e.closed)

    def estimate(self) -> float:
        return float(self.m) * float(self.closed_sum()) / float(self.r)


# ---- exact enumeration of one estimator under the IDEAL skip laws (for the pins) ---------------------------

class _Scripted:
    """Sampler whose outcomes are given; raises _Branch at the first call past the script."""

    __slots__ = ("script", "pos", "ev")

    def __init__(self, script):
        self.script, self.pos, self.ev = script, 0, 0

    def next_after(self, t):
        if t == 0:
            return 1
        if self.pos == len(self.script):
            raise _Branch(t)
        s = self.script[self.pos]
        self.pos += 1
        return s


class _Branch(Exception):
    def __init__(self, t):
        super().__init__(t)
        self.t = t


def enumerate_outcomes(stream):
    """Exact distribution of one estimator's final (f1, t1, f2, t2, chi, closed) after ``stream`` when every
    next_after(t) call has the ideal law P(T = s) = t/(s(s-1)), P(T > m) = t/m (outcomes beyond m are all
    equivalent: the event never happens).  Returns {outcome: Fraction}."""
    E = [normalize(u, v) for (u, v) in stream]
    m = len(E)
    out = {}

    def run(script, p):
        est = EventEst(_Scripted(script))
        deg = {}
        try:
            for t, e in enumerate(E, 1):
                for x in e:
                    deg[x] = deg.get(x, 0) + 1
                est.see(e, t, deg)
        except _Branch as b:
            t = b.t
            for s in range(t + 1, m + 1):
                run(script + [s], p * next_after_law(t, s))
            run(script + [m + 1], p * Fraction(t, m))  # T > m
            return
        key = (est.f1, est.t1, est.f2, est.t2, est.chi, est.closed)
        out[key] = out.get(key, Fraction(0)) + p

    run([], Fraction(1))
    return out
