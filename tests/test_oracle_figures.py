"""Pins from the paper's worked example (Figures 2, 4, 5) and App. B.

Fixtures under tests/golden/ carry their PAPER.md citations.
"""
import random

import numpy as np

from oracle import indexed, nbsi, rankall
from tcutil import golden_lines

L = "ABCDEF"
V = {ch: i for i, ch in enumerate(L)}


def _batch():
    line = golden_lines("fig4_rankall.txt")[0]
    assert line.startswith("W:")
    return [(V[e[0]], V[e[1]]) for e in line.split()[1:]]


def test_fig4_rankall_rows():
    """rankAll on W = <BC, CD, EF, BD, DF> reproduces Figure 4's rows I and II."""
    rows = {ln.split(":")[0]: ln.split(":")[1].split() for ln in golden_lines("fig4_rankall.txt")[1:]}
    Fp = rankall.rank_all(_batch())
    assert [L[e["src"]] for e in Fp] == rows["src"]
    assert [L[e["dst"]] for e in Fp] == rows["dst"]
    assert [str(e["pos"]) for e in Fp] == rows["pos"]
    assert [str(e["rank"]) for e in Fp] == rows["rank"]
    # the two ordering observations
    keys1 = [(e["src"], -e["pos"]) for e in Fp]
    keys2 = [(e["src"], e["rank"]) for e in Fp]
    assert keys1 == sorted(keys1) and keys2 == sorted(keys2)


def test_fig2_rank_table():
    """Definition Rank reproduces Figure 2's table."""
    W = _batch()
    for ln in golden_lines("fig2_rank.txt"):
        x, y, rk = ln.split()
        assert rankall.rank_def(W, V[x], V[y]) == int(rk), ln


def test_fig5_naming():
    """The naming system phi -> edge reproduces both Figure 5 tables with u = min
    endpoint (reading R1); the other orientation does NOT reproduce the right table."""
    W = _batch()
    Fp = rankall.rank_all(W)
    for ln in golden_lines("fig5_naming.txt"):
        f1, pos, *names = ln.split()
        p = int(pos) if int(pos) > 0 else -1
        got = rankall.name_substream(Fp, (V[f1[0]], V[f1[1]]), p)
        assert got == [frozenset((V[n[0]], V[n[1]])) for n in names], ln
    # orientation matters for CE: u = E gives EF first (reading R1)
    alt = rankall.name_substream(Fp, (V["C"], V["E"]), -1, u_first=V["E"])
    assert alt[0] == frozenset((V["E"], V["F"]))


def test_ranks_match_definition_random():
    """rankAll's scan-with-resets ranks == Definition Rank by brute force; Q1 ld/rd == rank(u->v)."""
    rnd = random.Random(7)
    for _ in range(40):
        n = rnd.randint(3, 9)
        pairs = [(a, b) for a in range(n) for b in range(a + 1, n)]
        rnd.shuffle(pairs)
        W = [tuple(rnd.sample(p, 2)) for p in pairs[: rnd.randint(1, len(pairs))]]
        Fp = rankall.rank_all(W)
        for e in Fp:
            assert e["rank"] == rankall.rank_def(W, e["src"], e["dst"])
        for x in range(n):
            for y in range(n):
                if x == y:
                    continue
                # the non-edge / old-edge case goes through the p = -1 footnote query
                pos = [i for i, w in enumerate(W, start=1) if set(w) == {x, y}]
                p = pos[0] if pos else -1
                ld, _ = rankall.ld_rd(Fp, (x, y), p)
                assert ld == rankall.rank_def(W, x, y)


def test_scan_with_resets_appB():
    """App. B: the sequential loop; SPEC-style example and a left fold of the
    printed operator agree with it.  The printed operator is NOT associative (reading R14)."""
    R = rankall.RESET
    assert rankall.scan_with_resets([1, 1, R, 1, 1]) == [0, 1, 2, 0, 1]
    assert rankall.scan_with_resets([R]) == [0]
    rnd = random.Random(3)
    for _ in range(200):
        A = [R if rnd.random() < 0.3 else 1 for _ in range(rnd.randint(1, 30))]
        acc, out = 0, []
        for a in A:  # exclusive left fold with the printed oplus, id = 0
            out.append(acc)
            acc = rankall.oplus(acc, a)
        assert out == rankall.scan_with_resets(A)
    # non-associativity counterexample: (1 (+) E) (+) 1 = 1  but  1 (+) (E (+) 1) = 2
    assert rankall.oplus(rankall.oplus(1, R), 1) != rankall.oplus(1, rankall.oplus(R, 1))


def test_worked_example_through_both_oracles():
    """The Figure 2 batch pushed after 3 old edges (CE, AC, AF: CE must be old per Fig. 5; the old
    dashed edges are not printed) through the brute-force and the bulk oracle: identical states."""
    old = [(V["C"], V["E"]), (V["A"], V["C"]), (V["A"], V["F"])]
    for seed in range(20):
        bo = nbsi.BruteOracle(64, seed)
        io = indexed.IndexedOracle(64, seed)
        for W in (old, _batch()):
            assert bo.push_batch(W) == 0 and io.push_batch(W) == 0
        a, b = bo.state(), io.state()
        for f in a:
            np.testing.assert_array_equal(a[f], b[f])
