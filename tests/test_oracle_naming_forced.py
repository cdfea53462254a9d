"""Forced-draw pins of the engine oracles' Step 2 naming and of the overflow guard.

* Figure 5 (naming system PAPER.md:761-767) through BOTH engine oracles: on the
  Figure 2 stream (old edges CE, AC, AF; W = <BC, CD, EF, BD, DF>), the draws are
  forced so that f1 becomes DC (fresh, Step 1 d1 = |E| + 1) or stays CE (retained), and Step 2's draw
  is d2 = chi^- + phi (reading R4: keep iff d2 < chi^-, else phi = d2 - chi^-).  The new f2 must be the
  edge Figure 5 names for phi: DC -> [DF, BD], CE -> [CD, CB, EF].  A wrong orientation (u = max), a
  reversed rank order or L/R swapped names a different edge and fails here.
* Reading R13: chi is kept exact in 64 bits and a batch after which some estimator's chi would exceed
  2^31 - 1 is rejected whole (TC_EOVERFLOW, nothing mutated); positions and m are unbounded (u64).
"""
import numpy as np
import pytest

from oracle import indexed, nbsi
from tcutil import golden_lines

L = "ABCDEF"
V = {ch: i for i, ch in enumerate(L)}
OLD = [(V["C"], V["E"]), (V["A"], V["C"]), (V["A"], V["F"])]


def _W():
    line = golden_lines("fig4_rankall.txt")[0]
    return [(V[e[0]], V[e[1]]) for e in line.split()[1:]]


def _cases():
    """(f1 name, position of f1 in W (1-based, 0 = old), [named edge per phi]) from the golden file."""
    out = []
    for ln in golden_lines("fig5_naming.txt"):
        f1, pos, *names = ln.split()
        out.append((f1, int(pos), names))
    return out


def _forced_draws(pos, phi):
    """Per batch (old, W): (d1, d2).  Old batch: f1 = CE (position 0); CE's only later old neighbour is
    AC, so chi^+ = 1 and d2 = 0 picks it (chi = 1).  Batch W (m_prev = 3): d1 = 3 + pos - 1 makes
    W[pos-1] the fresh f1 (chi^- = 0); d1 = 0 < m_prev retains CE (chi^- = 1).  d2 = chi^- + phi."""
    chi_minus = 0 if pos > 0 else 1
    d1_w = 3 + pos - 1 if pos > 0 else 0
    return [(0, 0), (d1_w, chi_minus + phi)]


def _edge(name):
    a, b = V[name[0]], V[name[1]]
    return (min(a, b), max(a, b))


@pytest.mark.parametrize("case", range(2))
def test_fig5_naming_through_engine_oracles(case):
    f1name, pos, names = _cases()[case]
    W = _W()
    EW = [nbsi.normalize(*e) for e in W]
    for phi, want in enumerate(names):
        draws = _forced_draws(pos, phi)
        # brute-force oracle (nbsi.py): the uniform(tag, n) hook returns the forced value
        bo = nbsi.BruteOracle(1, 0)
        for b, batch in enumerate((OLD, W)):
            d1, d2 = draws[b]

            def factory(i, bb, d1=d1, d2=d2):
                def uniform(tag, n):
                    v = d1 if tag == 1 else d2
                    assert 0 <= v < n, (tag, v, n)
                    return v
                return uniform
            assert bo.push_batch(batch, uniform_factory=factory) == 0
        # bulk oracle (indexed.c): rankAll + Q1/Q2 multisearch with the same forced draws
        io = indexed.IndexedOracle(1, 0)
        for b, batch in enumerate((OLD, W)):
            d1, d2 = draws[b]
            assert io.push_batch_forced(batch, [d1], [d2]) == 0
        for o in (bo, io):
            st = o.state()
            assert tuple(int(x) for x in st["r1"][0]) == _edge(f1name), f1name
            assert tuple(int(x) for x in st["r2"][0]) == _edge(want), (f1name, phi, want, st["r2"][0])
            assert int(st["p2"][0]) == 3 + EW.index(_edge(want))
            assert int(st["c"][0]) == (len(names) if pos else 1 + len(names))


def test_forced_draw_out_of_range_rejected():
    io = indexed.IndexedOracle(2, 0)
    before = io.state()
    assert io.push_batch_forced(OLD, [0, 3], [0, 0]) == nbsi.TC_EINVAL  # d1 = 3 is not < |E| + |W| = 3
    for f, v in before.items():
        np.testing.assert_array_equal(v, io.state()[f])
    assert io.counters() == (0, 0)


def _big_state():
    """Two estimators past any 32-bit position: m_prev = 2^33 + 5.  Estimator 0: f1 = (10, 11) at
    2^33, f2 = (11, 12) at 2^33 + 1, chi = 2^31 - 2.  Estimator 1: f1 = (20, 21) at 2^33 + 2, no f2."""
    M = (1 << 33) + 5
    return M, [((10, 11), 1 << 33, (11, 12), (1 << 33) + 1, (1 << 31) - 2, 0),
               ((20, 21), (1 << 33) + 2, nbsi.EMPTY_E, nbsi.EMPTY_P, 0, 0)]


def _both_with_state():
    M, ests = _big_state()
    bo = nbsi.BruteOracle(2, 9)
    io = indexed.IndexedOracle(2, 9)
    for i, (r1, p1, r2, p2, c, cl) in enumerate(ests):
        bo.ests[i] = nbsi.Est(r1=r1, p1=p1, r2=r2, p2=p2, c=c, closed=bool(cl))
        io.set_estimator(i, r1, p1, r2, p2, c, cl)
    bo.m, bo.b = M, 7
    io.set_counters(M, 7)
    return M, bo, io


def _push_both(bo, io, W, d1, d2):
    def factory(i, b):
        return lambda tag, n: d1[i] if tag == 1 else d2[i]
    return bo.push_batch(W, uniform_factory=factory), io.push_batch_forced(W, d1, d2)


def test_overflow_guard_chi_not_m():
    """chi^- + chi^+ > 2^31 - 1 rejects the batch in both oracles, state and counters unchanged; chi =
    2^31 - 1 exactly is accepted; m and positions beyond 2^32 are not limited (reading R13)."""
    M, bo, io = _both_with_state()
    before = io.state()
    # two later edges at f1 = (10, 11): chi = 2^31 - 2 + 2 = 2^31 > 2^31 - 1 -> TC_EOVERFLOW
    W = [(10, 30), (31, 11), (40, 41)]
    rb, ri = _push_both(bo, io, W, [0, 0], [0, 0])
    assert rb == ri == nbsi.TC_EOVERFLOW
    for o in (bo, io):
        for f, v in before.items():
            np.testing.assert_array_equal(v, o.state()[f], err_msg=f)
    assert io.counters() == (M, 7) and (bo.m, bo.b) == (M, 7)
    # one later edge: chi = 2^31 - 1 exactly -> accepted; estimator 1 takes a fresh f1 at 2^33 + 5 + 2
    W = [(10, 30), (40, 41), (20, 50)]
    rb, ri = _push_both(bo, io, W, [0, M + 2], [0, 0])
    assert rb == ri == 0
    a, b = bo.state(), io.state()
    for f in a:
        np.testing.assert_array_equal(a[f], b[f], err_msg=f)
    assert int(a["c"][0]) == (1 << 31) - 1 and int(a["p2"][0]) == (1 << 33) + 1  # kept f2 (d2 = 0 < chi^-)
    assert tuple(a["r1"][1]) == (20, 50) and int(a["p1"][1]) == M + 2 and int(a["c"][1]) == 0
    assert io.counters() == (M + 3, 8)


def test_huge_positions_philox_draws_agree():
    """With m_prev = 2^33 + 5 and real Philox draws the two oracles stay bit-identical: Step 1 bounds
    above 2^33 (64-bit Lemire), Step 2 draws over a growing chi and f2 positions above 2^32 for
    estimator 1 (estimator 0's f1 is never touched: its chi stays at 2^31 - 2)."""
    M, bo, io = _both_with_state()
    W = [(40, 41), (20, 50), (21, 51)]
    for k in range(40):  # Step 1 retains f1 (P(replace) = 3 / (m + 3)); every batch adds 2 to estimator 1's chi
        batch = [(a + 100 * k if a >= 30 else a, b_ + 100 * k if b_ >= 30 else b_) for a, b_ in W]
        assert bo.push_batch(batch) == 0 and io.push_batch(batch) == 0
    a, b = bo.state(), io.state()
    for f in a:
        np.testing.assert_array_equal(a[f], b[f], err_msg=f)
    assert int(a["c"][1]) == 80 and int(a["p2"][1]) > (1 << 33) and int(a["c"][0]) == (1 << 31) - 2
