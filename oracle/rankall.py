"""Literal rankAll, scan with resets, rank and the substream naming scheme.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  1-based positions, as in
the paper's figures.
"""
from __future__ import annotations

RESET = None  # the paper's "empty" element of App. B


def rank_def(W, x, y):
    """rank(x -> y) by Definition "Rank".

    If {x, y} = w_i for some i: |{j : x in w_j and j > i}|; otherwise deg_H(x).
    W is a list of 2-tuples, positions 1..|W|.
    """
    for i, w in enumerate(W, start=1):
        if set(w) == {x, y}:
            return sum(1 for j, wj in enumerate(W, start=1) if x in wj and j > i)
    return sum(1 for wj in W if x in wj)


def scan_with_resets(A):
    """App. B, the sequential loop verbatim:
    sum = 0; for i: out[i] = sum; if A[i] is empty: sum = 0 else sum += A[i]."""
    out, s = [], 0
    for a in A:
        out.append(s)
        s = 0 if a is RESET else s + a
    return out


def oplus(x, y):
    """App. B's operator on Z u {empty}, as printed:
    x+y if both non-empty; y if y non-empty; 0 otherwise."""
    if x is not RESET and y is not RESET:
        return x + y
    if y is not RESET:
        return y
    return 0


def rank_all(W):
    """rankAll(W) (Lemma rank-all proof).

    1. F: each w_i = {u, v} yields {src=u, dst=v, pos=i} and {src=v, dst=u, pos=i}.
    2. sort F by src, ties by decreasing pos.
    3. rank = scan with resets: the accumulator restarts at each new src
       (reading R14: the reset element sits on the last record of a src group,
       so the App. B loop emits 0 for the first record of the next group).
    Returns a list of dicts {src, dst, pos, rank} in the sorted order (Fig. 4).
    """
    F = []
    for i, (u, v) in enumerate(W, start=1):
        F.append(dict(src=u, dst=v, pos=i))
        F.append(dict(src=v, dst=u, pos=i))
    F.sort(key=lambda e: (e["src"], -e["pos"]))
    A = []
    for idx, e in enumerate(F):
        last_of_src = idx + 1 == len(F) or F[idx + 1]["src"] != e["src"]
        A.append(RESET if last_of_src else 1)
    for e, rk in zip(F, scan_with_resets(A)):
        e["rank"] = rk
    return F


def q1(Fp, u, p):
    """(Q1) "Given (u, p), locate an edge with src = u with the least pos larger or equal to p"
    (PAPER.md:809-811).  Returns the record or None."""
    cands = [e for e in Fp if e["src"] == u and e["pos"] >= p]
    return min(cands, key=lambda e: e["pos"]) if cands else None


def q2(Fp, u, a):
    """(Q2) "Given (u, a), locate an edge with src = u with the rank exactly equal to a"
    (PAPER.md:811-812)."""
    for e in Fp:
        if e["src"] == u and e["rank"] == a:
            return e
    return None


def ld_rd(Fp, f1, p):
    """ld = rank(u->v), rd = rank(v->u) through Q1.

    p = position of a fresh f1 in W; p = -1 for a retained f1 (footnote):
    the Q1 answer is then the arc with the largest rank at that src, and
    rank(u->v) of a non-edge is deg_W(u) = that rank + 1 (0 if u has no arc;
    reading R15).
    """
    u, v = f1

    def one(x):
        e = q1(Fp, x, p)
        if e is None:
            return 0
        return e["rank"] if p >= 0 else e["rank"] + 1

    return one(u), one(v)


def name_substream(Fp, f1, p, u_first=None):
    """The naming system phi -> edge of Gamma_W(f1) (Fig. 5).

    With u = min(f1) (reading R1) unless ``u_first`` overrides the orientation.
    Returns the list of undirected edges for phi = 0 .. chi^+ - 1.
    """
    u, v = (min(f1), max(f1)) if u_first is None else (u_first, (set(f1) - {u_first}).pop())
    ld, rd = ld_rd(Fp, (u, v), p)
    out = []
    for phi in range(ld + rd):
        src, a = (u, phi) if phi < ld else (v, phi - ld)
        e = q2(Fp, src, a)
        out.append(frozenset((e["src"], e["dst"])))
    return out
