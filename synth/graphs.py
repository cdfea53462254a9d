"""Seeded synthetic edge streams shaped like the paper's workloads.

The paper measures on SNAP graphs (Amazon, DBLP, LiveJournal, Orkut,
Friendster) and a 167 GB synthetic power-law graph (Table 1);
none of them is available here, so these generators stand in for their
shapes (BASELINE.json ``configs``):

* C1 Erdos-Renyi G(n=1000, m=20000)                         r=4096,  w=2048
* C2 R-MAT(0.57,0.19,0.19,0.05) scale 20, edge factor 16     r=2^20,  w=2^20
* C3 Chung-Lu gamma=2.1, n=3M, m=117M (Orkut-like)           r=2^22,  w=2^23
* C4 R-MAT scale 26 (~1B edges)                              r=2^24,  w=2^24
* C5 R-MAT scale 22, batch sweep                             r=2^22,  w=2^12..2^24

Every stream is a simple graph (self-loops and undirected duplicates
removed), vertex ids relabelled by a seeded permutation (R-MAT, Chung-Lu),
delivered in a seeded uniform-random order with each edge's orientation
flipped with probability 1/2.  Seeds: (graph, relabel, order, orientation)
derive from one integer through numpy's SeedSequence.
"""
from __future__ import annotations

import numpy as np

RMAT_ABCD = (0.57, 0.19, 0.19, 0.05)


def _rngs(seed: int):
    ss = np.random.SeedSequence(seed)
    g, rl, od, orient = ss.spawn(4)
    return (np.random.default_rng(g), np.random.default_rng(rl), np.random.default_rng(od),
            np.random.default_rng(orient))


def _dedup(u: np.ndarray, v: np.ndarray):
    """Drop self-loops and undirected duplicates; returns sorted unique (lo, hi)."""
    keep = u != v
    u, v = u[keep], v[keep]
    lo = np.minimum(u, v).astype(np.uint64)
    hi = np.maximum(u, v).astype(np.uint64)
    key = (lo << np.uint64(32)) | hi
    key.sort()
    if key.shape[0]:
        keep = np.empty(key.shape[0], bool)
        keep[0] = True
        np.not_equal(key[1:], key[:-1], out=keep[1:])
        key = key[keep]
    return (key >> np.uint64(32)).astype(np.uint32), (key & np.uint64(0xFFFFFFFF)).astype(np.uint32)


def finalize(lo: np.ndarray, hi: np.ndarray, r_order, r_orient, m: int | None = None) -> np.ndarray:
    """Random stream order (first m if given) and random orientation -> (m, 2) uint32."""
    perm = r_order.permutation(lo.shape[0])
    if m is not None:
        perm = perm[:m]
    a, b = lo[perm], hi[perm]
    flip = r_orient.random(a.shape[0]) < 0.5
    out = np.empty((a.shape[0], 2), dtype=np.uint32)
    out[:, 0] = np.where(flip, b, a)
    out[:, 1] = np.where(flip, a, b)
    return out


def er(n: int, m: int, seed: int = 1) -> np.ndarray:
    """Erdos-Renyi G(n, m): m distinct uniform pairs of [0, n), no loops."""
    rg, _, ro, rf = _rngs(seed)
    if m > n * (n - 1) // 2:
        raise ValueError("m too large for n")
    lo = np.empty(0, np.uint32)
    hi = np.empty(0, np.uint32)
    need = m
    while True:
        k = int(need * 1.3) + 16
        u = rg.integers(0, n, size=k, dtype=np.uint32)
        v = rg.integers(0, n, size=k, dtype=np.uint32)
        lo, hi = _dedup(np.concatenate([lo, u]), np.concatenate([hi, v]))
        if lo.shape[0] >= m:
            break
        need = m - lo.shape[0]
    # choose m of the unique pairs uniformly (random subset), then order/orient
    return finalize(lo, hi, ro, rf, m)


def rmat(scale: int, edge_factor: int = 16, seed: int = 1, abcd=RMAT_ABCD, chunk: int = 1 << 22) -> np.ndarray:
    """R-MAT(a, b, c, d) with 2^scale vertex ids and edge_factor * 2^scale draws (per-bit quadrant
    choice), loops and duplicates dropped, ids relabelled by a seeded permutation."""
    a, b, c, _ = abcd
    # quadrant thresholds on a 16-bit uniform (probabilities quantised to 1/65536)
    ta, tab, tabc = (np.uint16(round(x * 65536)) for x in (a, a + b, a + b + c))
    rg, rl, ro, rf = _rngs(seed)
    total = edge_factor << scale
    us, vs = [], []
    for start in range(0, total, chunk):
        k = min(chunk, total - start)
        u = np.zeros(k, np.uint32)
        v = np.zeros(k, np.uint32)
        for bit in range(scale):
            x = np.frombuffer(rg.bytes(2 * k), dtype=np.uint16)
            ubit = x >= tab
            vbit = ((x >= ta) & (x < tab)) | (x >= tabc)
            u |= ubit.astype(np.uint32) << np.uint32(bit)
            v |= vbit.astype(np.uint32) << np.uint32(bit)
        us.append(u)
        vs.append(v)
    u = np.concatenate(us)
    v = np.concatenate(vs)
    perm = rl.permutation(1 << scale).astype(np.uint32)
    lo, hi = _dedup(perm[u], perm[v])
    return finalize(lo, hi, ro, rf)


def chung_lu(n: int, m: int, gamma: float = 2.1, dmax: float = 66626.0, seed: int = 1) -> np.ndarray:
    """Chung-Lu power law: weights (i + i0)^(-1/(gamma-1)), i0 set so the largest expected degree
    is dmax; endpoints i.i.d. proportional to weight; loops/dups dropped until m unique edges."""
    rg, rl, ro, rf = _rngs(seed)
    i = np.arange(n, dtype=np.float64)
    ex = -1.0 / (gamma - 1.0)

    def maxdeg(i0):
        wts = (i + i0) ** ex
        return 2.0 * m * wts[0] / wts.sum()

    lo_i0, hi_i0 = 1e-3, 1e7
    for _ in range(200):  # bisection: maxdeg decreases in i0
        mid = (lo_i0 * hi_i0) ** 0.5
        if maxdeg(mid) > dmax:
            lo_i0 = mid
        else:
            hi_i0 = mid
    wts = (i + hi_i0) ** ex
    cdf = np.cumsum(wts)
    cdf /= cdf[-1]
    perm = rl.permutation(n).astype(np.uint32)
    lo = np.empty(0, np.uint32)
    hi = np.empty(0, np.uint32)
    need = m
    while True:
        k = int(need * 1.15) + 1024
        u = np.searchsorted(cdf, rg.random(k)).astype(np.uint32)
        v = np.searchsorted(cdf, rg.random(k)).astype(np.uint32)
        np.minimum(u, n - 1, out=u)
        np.minimum(v, n - 1, out=v)
        lo, hi = _dedup(np.concatenate([lo, perm[u]]), np.concatenate([hi, perm[v]]))
        if lo.shape[0] >= m:
            break
        need = m - lo.shape[0]
    return finalize(lo, hi, ro, rf, m)


def tiny_stream(n: int, m: int, seed: int) -> np.ndarray:
    """A small random simple-graph stream (m distinct pairs of [0, n)) for exhaustive tests."""
    return er(n, m, seed)


CONFIGS = {
    "C1": dict(kind="er", n=1000, m=20000, r=4096, w=2048,
               desc="Erdos-Renyi G(n=1000, m=20000); r=4096, w=2048"),
    "C2": dict(kind="rmat", scale=20, edge_factor=16, r=1 << 20, w=1 << 20,
               desc="R-MAT(0.57,0.19,0.19,0.05) scale 20, edge factor 16 (~15.7M unique); r=2^20, w=2^20"),
    "C3": dict(kind="chung_lu", n=3_000_000, m=117_000_000, gamma=2.1, r=1 << 22, w=1 << 23,
               desc="Chung-Lu gamma=2.1, n=3M, m=117M; r=2^22, w=2^23"),
    "C4": dict(kind="rmat", scale=26, edge_factor=16, r=1 << 24, w=1 << 24,
               desc="R-MAT scale 26 (~1B unique); r=2^24, w=2^24"),
    "C5": dict(kind="rmat", scale=22, edge_factor=16, r=1 << 22, w=1 << 20,
               desc="R-MAT scale 22 (~64M unique); r=2^22, w swept 2^12..2^24"),
}


def config_stream(name: str, seed: int = 1) -> np.ndarray:
    """The stream of a BASELINE.json config.  C1 comes from the numpy generator above; C2-C5 from the
    native counter-based generator (synth/gen.c: same recipe, seconds instead of minutes at 10^8-10^9
    edges)."""
    cfg = CONFIGS[name]
    if cfg["kind"] == "er":
        return er(cfg["n"], cfg["m"], seed)
    from . import native
    if cfg["kind"] == "rmat":
        return native.rmat(cfg["scale"], cfg["edge_factor"], seed)
    if cfg["kind"] == "chung_lu":
        return native.chung_lu(cfg["n"], cfg["m"], cfg["gamma"], seed=seed)
    raise KeyError(name)
