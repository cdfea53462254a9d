"""Pins for the oracle's randomness (readings R7, R8).

* Philox4x32-10 (Python and C oracle implementations) == cuRAND's own
  ``curand_Philox4x32_10`` host path (a third-party routine), element by element.
* Lemire's bounded uniform: closed forms (n = 2^k is a shift, n = 1 is 0, n = 3
  rejects exactly x = 0) and the retry path.
"""
import os
import shutil
import subprocess
import tempfile

import numpy as np
import pytest

from oracle import indexed, rng

HELPER = os.path.join(os.path.dirname(__file__), "helpers", "curand_philox_host.cu")


@pytest.fixture(scope="module")
def curand_bin():
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available for the cuRAND host pin")
    d = tempfile.mkdtemp()
    exe = os.path.join(d, "cph")
    subprocess.check_call([nvcc, "-Wno-deprecated-gpu-targets", "-o", exe, HELPER], cwd=d)
    return exe


def test_philox_vs_curand(curand_bin):
    g = np.random.default_rng(11)
    cases = g.integers(0, 2**32, size=(500, 6), dtype=np.uint64)
    cases[:4] = [[0, 0, 0, 0, 0, 0], [2**32 - 1] * 6, [1, 0, 0, 0, 0, 0], [0, 0, 0, 0x10001, 42, 0]]
    inp = "\n".join(" ".join(str(int(x)) for x in row) for row in cases) + "\n"
    out = subprocess.run([curand_bin], input=inp, capture_output=True, text=True, check=True).stdout
    ref = [tuple(int(x) for x in ln.split()) for ln in out.strip().splitlines()]
    assert len(ref) == len(cases)
    vec = rng.philox4x32_10_np(*[cases[:, j] for j in range(6)])
    for t, row in enumerate(cases):
        ctr, key = tuple(int(x) for x in row[:4]), tuple(int(x) for x in row[4:])
        assert rng.philox4x32_10(ctr, key) == ref[t]
        assert indexed.philox(ctr, key) == ref[t]
        assert tuple(int(v[t]) for v in vec) == ref[t]


def test_lemire_closed_forms():
    g = np.random.default_rng(5)
    no_retry = lambda t: pytest.fail("unexpected retry")  # noqa: E731
    for x in [int(v) for v in g.integers(0, 2**63, size=200, dtype=np.uint64)] + [0, 1, 2**64 - 1]:
        for k in range(0, 64):
            assert rng.lemire(1 << k, x, no_retry) == x >> (64 - k)  # n = 2^k: a shift, never rejects
        assert rng.lemire(1, x, no_retry) == 0
    # n = 3: threshold (2^64 - 3) mod 3 = 1, so only x = 0 (low64(3x) = 0) is rejected
    assert rng.lemire(3, 2**64 - 1, no_retry) == 2
    assert rng.lemire(3, 1, no_retry) == 0
    assert rng.lemire(3, 0, lambda t: [None, 0, 2**63][t]) == 1  # retries: 0 rejected again, then 2^63
    # general n: floor(x*n / 2^64) whenever not rejected
    for n in (5, 7, 1000, 2**40 + 3):
        thr = (2**64 - n) % n
        for x in (int(v) for v in g.integers(0, 2**63, size=100, dtype=np.uint64)):
            if (x * n) % 2**64 >= thr:
                assert rng.lemire(n, x, no_retry) == (x * n) >> 64


def test_lemire_c_matches_python():
    g = np.random.default_rng(9)
    for _ in range(300):
        n = int(g.integers(1, 2**62))
        x = int(g.integers(0, 2**63))
        seed, i, b = int(g.integers(0, 2**63)), int(g.integers(0, 2**40)), int(g.integers(0, 100))
        hook = rng.PhiloxDraws(seed, i, b)
        py = rng.lemire(n, x, lambda t: rng.words64(hook._block(rng.STEP1_RETRY_BASE + t))[0])
        assert indexed.lib().orc_lemire_words(n, x, seed, i, b, rng.STEP1_RETRY_BASE) == py
    # a forced rejection: n = 3, x = 0 must take the retry word (ctr.w = 0x10001, low 64 bits)
    seed, i, b = 42, 7, 3
    hook = rng.PhiloxDraws(seed, i, b)
    w1 = rng.words64(hook._block(rng.STEP1_RETRY_BASE + 1))[0]
    assert indexed.lib().orc_lemire_words(3, 0, seed, i, b, rng.STEP1_RETRY_BASE) == (w1 * 3) >> 64


def test_batch_words_vectorised():
    ids = np.array([0, 1, 2**32 + 5, 2**40 - 1], dtype=np.uint64)
    lo, hi = rng.batch_words(123456789012345, ids, 77)
    for t, i in enumerate(ids):
        blk = rng.philox4x32_10((int(i) & 0xFFFFFFFF, int(i) >> 32, 77, 0),
                                (123456789012345 & 0xFFFFFFFF, 123456789012345 >> 32))
        assert (int(lo[t]), int(hi[t])) == rng.words64(blk)
