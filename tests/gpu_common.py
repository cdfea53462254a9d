"""Helpers for the -m gpu parity tests: run the CUDA path and the oracle on the same seeded input."""
import numpy as np

FIELDS = ("r1", "p1", "r2", "p2", "c", "closed")


def gpu_run(stream, r, seed, w, first=0, count=None, device_input=False, **kw):
    from paper_1308_2166_b200 import TriangleCounter
    tc = TriangleCounter(r, seed, first=first, count=count, **kw)
    if device_input:
        import torch
        dev = torch.from_numpy(np.ascontiguousarray(stream).view(np.int32)).cuda()
    for k in range(0, len(stream), w):
        if device_input:
            tc.push_batch(dev[k:k + w])
        else:
            tc.push_batch(stream[k:k + w])
    return tc


def oracle_run(stream, r, seed, w, first=0, count=None):
    from oracle.indexed import IndexedOracle
    o = IndexedOracle(r, seed, first, count)
    for k in range(0, len(stream), w):
        assert o.push_batch(stream[k:k + w]) == 0
    return o


def assert_states_equal(a, b, where=""):
    for f in FIELDS:
        if not np.array_equal(a[f], b[f]):
            bad = np.nonzero((a[f] != b[f]).reshape(len(a[f]), -1).any(axis=1))[0]
            i = int(bad[0])
            raise AssertionError(f"{where}: field {f} differs at {len(bad)} estimators; first local id {i}: "
                                 + ", ".join(f"{g}={a[g][i]}/{b[g][i]}" for g in FIELDS))


def check_properties(stream, st, m):
    """NBSI properties that hold at any size, checked vectorised against the stream prefix."""
    E = np.sort(stream[:m], axis=1).astype(np.uint64)
    keys = (E[:, 0] << np.uint64(32)) | E[:, 1]
    order = np.argsort(keys)
    skeys = keys[order]
    p1 = st["p1"].astype(np.int64)
    assert (p1 >= 0).all() and (p1 < m).all()
    assert np.array_equal(E[p1].astype(np.uint32), st["r1"])
    has2 = st["c"] > 0
    assert np.array_equal(has2, st["p2"] != np.uint64(2**64 - 1))
    p2 = st["p2"][has2].astype(np.int64)
    assert (p2 > p1[has2]).all() and (p2 < m).all()
    assert np.array_equal(E[p2].astype(np.uint32), st["r2"][has2])
    r1, r2 = st["r1"][has2].astype(np.int64), st["r2"][has2].astype(np.int64)
    share = (r1[:, :1] == r2).any(1) | (r1[:, 1:] == r2).any(1)
    assert share.all()
    # closed <=> the closing edge occurs after f2
    x = np.where((r1[:, 0:1] == r2).any(1), r1[:, 1], r1[:, 0])
    z = np.where((r2[:, 0:1] == r1).any(1), r2[:, 1], r2[:, 0])
    lo, hi = np.minimum(x, z).astype(np.uint64), np.maximum(x, z).astype(np.uint64)
    q = (lo << np.uint64(32)) | hi
    idx = np.searchsorted(skeys, q)
    idx = np.minimum(idx, len(skeys) - 1)
    found = skeys[idx] == q
    pos = np.where(found, order[idx], -1)
    closing = found & (pos > p2)
    assert np.array_equal(closing, st["closed"][has2].astype(bool))
    assert not st["closed"][~has2].any()
    # chi == |Gamma_S(f1)|: arcs at u or v strictly after p1 (NBSI clause 2)
    arcs_v = np.concatenate([E[:, 0], E[:, 1]])
    arcs_p = np.concatenate([np.arange(m, dtype=np.uint64)] * 2)
    akeys = np.sort((arcs_v << np.uint64(32)) | arcs_p)
    u = st["r1"][:, 0].astype(np.uint64)
    v = st["r1"][:, 1].astype(np.uint64)
    pp = st["p1"].astype(np.uint64)
    top = np.uint64(0xFFFFFFFF)

    def after(x):
        return (np.searchsorted(akeys, (x << np.uint64(32)) | top, side="right")
                - np.searchsorted(akeys, (x << np.uint64(32)) | pp, side="right"))

    assert np.array_equal(after(u) + after(v), st["c"].astype(np.int64))
