"""The seeded input generators (synth/, inputs only): determinism independent of the thread count, simple
graphs, and the shapes of the BASELINE.json configs."""
import os
import subprocess
import sys

import numpy as np

from synth import native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _simple(s):
    assert (s[:, 0] != s[:, 1]).all()
    k = np.sort(s, 1).astype(np.uint64)
    key = (k[:, 0] << np.uint64(32)) | k[:, 1]
    assert len(np.unique(key)) == len(s)


def test_rmat_deterministic_across_thread_counts():
    code = ("import sys, hashlib; sys.path.insert(0, %r); from synth import native; "
            "s = native.rmat(14, 16, 5); print(len(s), hashlib.sha1(s.tobytes()).hexdigest())" % ROOT)
    outs = set()
    for nt in ("1", "3", "8"):
        env = dict(os.environ, OMP_NUM_THREADS=nt)
        outs.add(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                                check=True).stdout)
    assert len(outs) == 1


def test_rmat_shape():
    s = native.rmat(16, 16, 3)
    _simple(s)
    assert 0.80 * (16 << 16) < len(s) < (16 << 16)  # ~13% duplicates at this skew and density
    assert s.max() < (1 << 16)
    deg = np.bincount(s.ravel().astype(np.int64), minlength=1 << 16)
    assert deg.max() > 50 * deg.mean()  # power-law hubs
    assert 0.4 < np.mean(s[:, 0] < s[:, 1]) < 0.6  # random orientation
    assert not np.array_equal(native.rmat(16, 16, 4), s)


def test_chung_lu_shape():
    n, m = 200_000, 2_000_000
    s = native.chung_lu(n, m, 2.1, dmax=5000.0, seed=2)
    _simple(s)
    assert len(s) == m and s.max() < n
    deg = np.bincount(s.ravel().astype(np.int64), minlength=n)
    assert 3000 < deg.max() < 7000  # the largest expected degree is dmax
    # random stream order: the first and second half have the same degree profile of their endpoints
    a = np.bincount(s[: m // 2].ravel().astype(np.int64), minlength=n)
    b = np.bincount(s[m // 2:].ravel().astype(np.int64), minlength=n)
    assert abs(int(a.max()) - int(b.max())) < 0.1 * deg.max()
