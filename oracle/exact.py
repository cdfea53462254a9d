"""Ground truth for the oracle pins: tau, Gamma_S, C(t), and exact enumeration.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Definitions (§2): G simple undirected; the stream order is
a total order on E; Gamma_S(e) = {f in E : f shares exactly one vertex with e
and f >_S e}; T(G) the triangles, tau = |T(G)|; C(t) = |Gamma_S(f)| for f the
first edge of t in stream order.
"""
from __future__ import annotations

from collections import defaultdict
from fractions import Fraction

from . import nbsi


def norm_stream(stream):
    return [nbsi.normalize(u, v) for (u, v) in stream]


def triangles(stream):
    """All triangles of the graph, each as a frozenset of its 3 edges (brute force via adjacency)."""
    E = norm_stream(stream)
    adj = defaultdict(set)
    for (u, v) in E:
        adj[u].add(v)
        adj[v].add(u)
    out = []
    for (u, v) in E:
        for w in adj[u] & adj[v]:
            if w > v:  # u < v < w: each triangle once
                out.append(frozenset({(u, v), nbsi.normalize(u, w), nbsi.normalize(v, w)}))
    return out


def triangle_count(stream):
    """tau = |T(G)| by the adjacency-matrix identity tau = sum((A @ A) * A) / 6
    (each triangle is 6 closed walks of length 3 through its edges); scipy sparse matmul is the library
    step.  For graphs whose wedge count sum_v deg(v)^2 fits memory (the accuracy study's ground truth is
    the GPU counter; this is its oracle at test sizes)."""
    import numpy as np
    import scipy.sparse as sp
    E = np.asarray(stream, dtype=np.int64).reshape(-1, 2)
    if len(E) == 0:
        return 0
    ids, inv = np.unique(E.ravel(), return_inverse=True)
    inv = inv.reshape(-1, 2)
    n = len(ids)
    rows = np.concatenate([inv[:, 0], inv[:, 1]])
    cols = np.concatenate([inv[:, 1], inv[:, 0]])
    A = sp.csr_matrix((np.ones(len(rows), dtype=np.int64), (rows, cols)), shape=(n, n))
    return int((A @ A).multiply(A).sum()) // 6


def gamma_sizes(stream):
    """|Gamma_S(e_i)| for every stream position i (definition at)."""
    E = norm_stream(stream)
    later = defaultdict(int)  # occurrences of a vertex strictly after the current position
    out = [0] * len(E)
    for i in range(len(E) - 1, -1, -1):
        u, v = E[i]
        out[i] = later[u] + later[v]
        later[u] += 1
        later[v] += 1
    return out


def gamma_brute(stream, i):
    """|Gamma_S(e_i)| straight from the definition (quadratic; tiny inputs)."""
    E = norm_stream(stream)
    e = set(E[i])
    return sum(1 for j in range(i + 1, len(E)) if len(e & set(E[j])) == 1)


def C_values(stream):
    """C(t) for every triangle t."""
    E = norm_stream(stream)
    pos = {e: i for i, e in enumerate(E)}
    g = gamma_sizes(stream)
    return [g[min(pos[e] for e in t)] for t in triangles(stream)]


def moments(stream):
    """(tau, sum_t C(t), m): E[X] = tau (Lemma unbiased-est) and, from Claim
    discovery-prob, X = m*C(t) w.p. 1/(m*C(t)) per triangle t, so
    E[X^2] = m * sum_t C(t)."""
    Cs = C_values(stream)
    return len(Cs), sum(Cs), len(stream)


# ---------------------------------------------------------------------------
# Exact enumeration of one estimator's outcome tree (rational probabilities)
# ---------------------------------------------------------------------------

def _freeze(est):
    return (est.r1, est.p1, est.r2, est.p2, est.c, est.closed)


def _thaw(t):
    return nbsi.Est(r1=t[0], p1=t[1], r2=t[2], p2=t[3], c=t[4], closed=t[5])


def _branches(state, E_W, E_lo, E_hi, m_prev):
    """All outcomes of one estimator's batch update, each with its exact probability.

    Drives nbsi.step1..3 with a replaying ``uniform`` hook: a depth-first walk
    over every sequence of draw outcomes, each draw over [0, n) weighted 1/n.
    """
    out = []
    stack = [[]]
    while stack:
        prefix = stack.pop()
        calls = []

        def hook(tag, n, prefix=prefix, calls=calls):
            t = len(calls)
            calls.append(n)
            return prefix[t] if t < len(prefix) else 0

        est = _thaw(state)
        nbsi.step1_level1(est, E_W, m_prev, hook)
        nbsi.step2_level2(est, E_W, E_lo, E_hi, m_prev, hook)
        nbsi.step3_closing(est, E_W, m_prev)
        full = prefix + [0] * (len(calls) - len(prefix))
        p = Fraction(1)
        for n in calls:
            p /= n
        out.append((_freeze(est), p))
        for t in range(len(prefix), len(calls)):
            for alt in range(1, calls[t]):
                stack.append(full[:t] + [alt])
    return out


def enumerate_distribution(stream, batch_sizes):
    """Exact distribution over final states (r1, p1, r2, p2, c, closed) of ONE estimator
    after feeding ``stream`` in consecutive batches of the given sizes."""
    import numpy as np
    assert sum(batch_sizes) == len(stream)
    dist = {_freeze(nbsi.Est()): Fraction(1)}
    m_prev = 0
    for s in batch_sizes:
        W = stream[m_prev:m_prev + s]
        E_W = norm_stream(W)
        E_lo = np.array([e[0] for e in E_W], dtype=np.int64)
        E_hi = np.array([e[1] for e in E_W], dtype=np.int64)
        new = defaultdict(Fraction)
        for st, pr in dist.items():
            for st2, q in _branches(st, E_W, E_lo, E_hi, m_prev):
                new[st2] += pr * q
        dist = dict(new)
        m_prev += s
    return dist


def dist_moments(dist, m):
    """(E[X], E[X^2]) of X = c*m if closed else 0 under an exact distribution."""
    ex = Fraction(0)
    ex2 = Fraction(0)
    for st, pr in dist.items():
        x = st[4] * m if st[5] else 0
        ex += pr * x
        ex2 += pr * x * x
    return ex, ex2
