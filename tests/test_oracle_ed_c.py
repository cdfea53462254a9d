"""oracle/ed.c (event walk per estimator, OpenMP) == oracle/ed.py (plain per-edge rule, pinned by exact
enumeration in test_oracle_ed.py), field by field, on random streams at every prefix of a random batching;
the C sampler equals the Python sampler word for word."""
import random

import numpy as np
import pytest

from oracle import ed, edc
from synth import er, rmat


def _eq(a, b, where):
    for f in a:
        np.testing.assert_array_equal(a[f], b[f], err_msg=f"{where}: {f}")


def test_sampler_same_words():
    rnd = random.Random(1)
    for _ in range(400):
        t = rnd.choice([0, 1, 2, 3, rnd.randrange(1, 1000), rnd.randrange(1, 1 << 31), (1 << 31) - 1])
        i, seed, ev = rnd.randrange(1 << 40), rnd.randrange(1 << 64), rnd.randrange(64)
        w = ed.WordStream(seed, i, ev)
        s = ed.next_after(t, w)
        assert edc.next_after(t, i, seed, ev) == (s, w.ev), (t, i, seed, ev)


@pytest.mark.parametrize("seed", range(4))
def test_c_equals_plain_every_prefix(seed):
    s = er(40, 260, seed + 7) if seed % 2 == 0 else [tuple(e) for e in rmat(7, 3, seed).tolist()][:260]
    r = 80
    a = ed.EventOracle(r, seed)
    b = edc.EventOracleC(r, seed)
    rnd = random.Random(seed)
    k = 0
    while k < len(s):
        w = rnd.choice([1, 5, 31, 90])
        W = s[k:k + w]
        assert a.push_batch(W) == 0 and b.push_batch(W) == 0
        k += len(W)
        _eq(a.state(), b.state(), f"prefix {k}")
    assert a.closed_sum() == b.closed_sum() and a.estimate() == b.estimate()


def test_c_equals_plain_sharded_ids():
    s = er(30, 200, 3)
    a = ed.EventOracle(1 << 40, 9, first=(1 << 40) - 50, count=50)
    b = edc.EventOracleC(1 << 40, 9, first=(1 << 40) - 50, count=50)
    assert a.push_batch(s) == 0 and b.push_batch(s) == 0
    _eq(a.state(), b.state(), "high ids")


def test_c_rejections():
    b = edc.EventOracleC(10, 1)
    assert b.push_batch([(1, 2), (2, 1)]) == -4
    assert b.push_batch([(3, 3)]) == -3
    assert b.m == 0


def test_c_nbsi_midsize():
    """NBSI clauses by brute force on a 3000-edge power-law prefix (C oracle only)."""
    from test_oracle_exact import _check_nbsi
    s = [tuple(e) for e in rmat(10, 4, 5).tolist()][:3000]
    b = edc.EventOracleC(300, 2)
    assert b.push_batch(s) == 0
    st = b.state()
    _check_nbsi(s, st)
    assert (st["J"] > len(s)).all()
