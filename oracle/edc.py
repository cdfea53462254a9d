"""ctypes front end of oracle/ed.c: the event-driven oracle walked estimator by estimator (OpenMP).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Same rule and same random words as oracle/ed.py (reading
R17); the state after a prefix is computed from the prefix alone (the mode is batch-invariant), so a push only
validates and appends.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from . import ed
from .nbsi import EMPTY_P, EMPTY_V, TC_EOVERFLOW, TC_OK, validate_batch

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "ed.c")
LIB = os.path.join(HERE, "liboracle_ed.so")

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=gnu11", "-Wall",
                               "-o", tmp, SRC])
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        u64, vp = C.c_uint64, C.c_void_p
        L.orc_ed_run.restype = C.c_int
        L.orc_ed_run.argtypes = [vp, u64, u64, u64, u64, vp, vp, vp, vp, vp, vp, vp]
        L.orc_ed_next_after.restype = C.c_uint32
        L.orc_ed_next_after.argtypes = [u64, u64, u64, u64, C.POINTER(u64)]
        L.orc_ed_threads.restype = C.c_int
        _lib = L
    return _lib


def next_after(t: int, i: int, seed: int, ev: int = 0):
    """(next_after(t), words used after) for estimator i starting at word ev."""
    out = C.c_uint64(0)
    s = lib().orc_ed_next_after(t, i, seed, ev, C.byref(out))
    return int(s), int(out.value)


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class EventOracleC:
    """Estimators [first, first + count) of r, event-driven mode."""

    def __init__(self, r: int, seed: int, first: int = 0, count: int | None = None):
        if r <= 0:
            raise ValueError("r must be >= 1")
        self.r, self.seed, self.first = r, seed, first
        self.count = r - first if count is None else count
        self.parts = []
        self.m = 0
        self.deg = {}
        self._cache = None

    def push_batch(self, W, validate: bool = True) -> int:
        W = np.ascontiguousarray(np.asarray(W, dtype=np.uint32).reshape(-1, 2))
        if len(W) == 0:
            return TC_OK
        if validate:
            code = validate_batch([tuple(map(int, e)) for e in W])
            if code != TC_OK:
                return code
            v, c = np.unique(W.ravel(), return_counts=True)
            if any(self.deg.get(int(x), 0) + int(d) > ed.DEG_MAX for x, d in zip(v, c)):
                return TC_EOVERFLOW
            for x, d in zip(v.tolist(), c.tolist()):
                self.deg[x] = self.deg.get(x, 0) + d
        self.parts.append(W)
        self.m += len(W)
        self._cache = None
        return TC_OK

    def _run(self):
        if self._cache is None:
            s = np.ascontiguousarray(np.concatenate(self.parts) if self.parts else np.zeros((0, 2), np.uint32))
            n = self.count
            t1, t2, chi, J, K = (np.zeros(n, np.uint32) for _ in range(5))
            closed = np.zeros(n, np.uint8)
            ev = np.zeros(n, np.uint64)
            rc = lib().orc_ed_run(_p(s), self.m, self.seed, self.first, n, _p(t1), _p(t2), _p(chi), _p(closed),
                                  _p(J), _p(K), _p(ev))
            if rc != 0:
                raise MemoryError("orc_ed_run")
            self._cache = (s, t1, t2, chi, closed, J, K, ev)
        return self._cache

    def state(self):
        s, t1, t2, chi, closed, J, K, ev = self._run()
        E = np.sort(s, axis=1) if len(s) else s

        def edge(t):
            out = np.full((len(t), 2), EMPTY_V, np.uint32)
            ok = t > 0
            out[ok] = E[t[ok].astype(np.int64) - 1]
            return out

        def pos(t):
            return np.where(t > 0, t.astype(np.uint64) - np.uint64(1), np.uint64(EMPTY_P))

        return dict(r1=edge(t1), p1=pos(t1), r2=edge(t2), p2=pos(t2), c=chi.copy(), closed=closed.copy(),
                    J=J.copy(), K=K.copy(), ev=ev.copy())

    def closed_sum(self) -> int:
        _, _, _, chi, closed, _, _, _ = self._run()
        return int(chi[closed == 1].astype(np.uint64).sum())

    def estimate(self) -> float:
        return float(self.m) * float(self.closed_sum()) / float(self.r)


def threads() -> int:
    return int(lib().orc_ed_threads())
