"""Oracle randomness: Philox4x32-10 and Lemire's bounded uniform integer.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper is silent on how random bits are produced; it only notes that the
sequential and the parallel algorithm "produce the exact same answer given the
same sequence of random bits" (§5 "Baseline").  The mapping
below is DESIGN.md reading R7 (draw placement) and R8 (uniform method):

* one Philox4x32-10 call per (estimator i, non-empty batch b):
      ctr = (i mod 2^32, i >> 32, b, 0),  key = (seed mod 2^32, seed >> 32)
      out = (x, y, z, w)
      x_lo = x | y << 32   -- feeds Step 1's draw randInt(|W| + |E|)
      x_hi = z | w << 32   -- feeds Step 2's draw over chi^- + chi^+  
* Lemire's multiply-shift with rejection U(x, n) = floor(x * n / 2^64);
  on rejection the t-th retry word (t = 1, 2, ...) comes from the same
  counter with ctr.w = 0x10000 + t (Step 1) or 0x20000 + t (Step 2), using
  the low 64 bits of that block.

Philox4x32-10 itself is the published generator (Salmon et al., SC'11); the
constants and the round function are written out here from its definition
and pinned in tests against cuRAND's host implementation
(``curand_Philox4x32_10``) -- a third-party routine, not this code.
"""
from __future__ import annotations

import numpy as np

M0 = 0xD2511F53
M1 = 0xCD9E8D57
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK32 = 0xFFFFFFFF
MASK64 = (1 << 64) - 1

STEP1_RETRY_BASE = 0x10000
STEP2_RETRY_BASE = 0x20000


def philox4x32_10(ctr, key):
    """Philox4x32-10 on one 128-bit counter; ctr = 4 x u32, key = 2 x u32 (Python ints)."""
    c0, c1, c2, c3 = (int(v) & MASK32 for v in ctr)
    k0, k1 = (int(v) & MASK32 for v in key)
    for rnd in range(10):
        if rnd:
            k0 = (k0 + W0) & MASK32
            k1 = (k1 + W1) & MASK32
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> 32, p0 & MASK32
        hi1, lo1 = p1 >> 32, p1 & MASK32
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return (c0, c1, c2, c3)


def philox4x32_10_np(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10: every argument is a uint32 array (or scalar), broadcast together."""
    c0, c1, c2, c3 = (np.asarray(v, dtype=np.uint64) & np.uint64(MASK32) for v in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=np.uint64) & np.uint64(MASK32)
    k1 = np.asarray(k1, dtype=np.uint64) & np.uint64(MASK32)
    m32 = np.uint64(MASK32)
    s32 = np.uint64(32)
    for rnd in range(10):
        if rnd:
            k0 = (k0 + np.uint64(W0)) & m32
            k1 = (k1 + np.uint64(W1)) & m32
        p0 = np.uint64(M0) * c0
        p1 = np.uint64(M1) * c2
        c0, c1, c2, c3 = ((p1 >> s32) ^ c1 ^ k0, p1 & m32, (p0 >> s32) ^ c3 ^ k1, p0 & m32)
    return (c0.astype(np.uint32), c1.astype(np.uint32), c2.astype(np.uint32), c3.astype(np.uint32))


def words64(block):
    """(x, y, z, w) -> (x | y<<32, z | w<<32)."""
    x, y, z, w = block
    return (int(x) | (int(y) << 32), int(z) | (int(w) << 32))


def lemire(n, first, retry):
    """Uniform integer in [0, n) from 64-bit words (Lemire 2019, multiply-shift with rejection).

    ``first`` is the first 64-bit word; ``retry(t)`` returns the t-th retry word.
    p = x*n (128-bit); reject while low64(p) < (2^64 - n) mod n; return high64(p).
    """
    if n <= 0:
        raise ValueError("uniform over an empty range")
    x = first
    p = x * n
    lo = p & MASK64
    if lo < n:
        thresh = ((1 << 64) - n) % n
        t = 0
        while lo < thresh:
            t += 1
            x = retry(t)
            p = x * n
            lo = p & MASK64
    return p >> 64


class PhiloxDraws:
    """The production ``uniform(tag, n)`` hook for one (estimator, batch) pair.

    tag 1 = Step 1 (level-1 reservoir), tag 2 = Step 2 (level-2 choice).
    """

    __slots__ = ("i", "b", "seed", "_words")

    def __init__(self, seed: int, i: int, b: int, words=None):
        self.seed, self.i, self.b = seed, i, b
        self._words = words  # optional precomputed (x_lo, x_hi)

    def _block(self, w: int):
        return philox4x32_10((self.i & MASK32, (self.i >> 32) & MASK32, self.b & MASK32, w),
                             (self.seed & MASK32, (self.seed >> 32) & MASK32))

    def __call__(self, tag: int, n: int) -> int:
        if self._words is None:
            self._words = words64(self._block(0))
        first = self._words[0] if tag == 1 else self._words[1]
        base = STEP1_RETRY_BASE if tag == 1 else STEP2_RETRY_BASE
        return lemire(n, first, lambda t: words64(self._block(base + t))[0])


def batch_words(seed: int, ids: np.ndarray, b: int):
    """Vectorised first words (x_lo, x_hi) for estimator ids ``ids`` in batch ``b`` (uint64 arrays)."""
    ids = np.asarray(ids, dtype=np.uint64)
    o = philox4x32_10_np(ids & np.uint64(MASK32), ids >> np.uint64(32), np.uint64(b & MASK32),
                         np.uint64(0), np.uint64(seed & MASK32), np.uint64((seed >> 32) & MASK32))
    x = [v.astype(np.uint64) for v in o]
    return (x[0] | (x[1] << np.uint64(32)), x[2] | (x[3] << np.uint64(32)))
