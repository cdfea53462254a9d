"""ctypes front end for oracle/indexed.c (the paper's bulk algorithm on the CPU, OpenMP).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  ``build()`` compiles the C
file with gcc; it is also called by ``__graft_entry__.build()`` (building the
checker is not using it).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "indexed.c")
LIB = os.path.join(HERE, "liboracle_indexed.so")

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-Wall",
                               "-o", tmp, SRC])
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        u64, u32, vp = C.c_uint64, C.c_uint32, C.c_void_p
        L.orc_create.restype = vp
        L.orc_create.argtypes = [u64, u64, u64, u64]
        L.orc_destroy.argtypes = [vp]
        L.orc_push_batch.restype = C.c_int
        L.orc_push_batch.argtypes = [vp, vp, u64]
        L.orc_get_state.argtypes = [vp, vp, vp, vp, vp, vp, vp]
        L.orc_closed_sum.restype = u64
        L.orc_closed_sum.argtypes = [vp]
        L.orc_counters.argtypes = [vp, C.POINTER(u64), C.POINTER(u32)]
        L.orc_philox.argtypes = [vp, vp, vp]
        L.orc_lemire_words.restype = u64
        L.orc_lemire_words.argtypes = [u64, u64, u64, u64, u32, u32]
        L.orc_threads.restype = C.c_int
        L.orc_push_batch_forced.restype = C.c_int
        L.orc_push_batch_forced.argtypes = [vp, vp, u64, vp, vp]
        L.orc_set_estimator.argtypes = [vp, u64, vp, u64, vp, u64, u32, C.c_uint8]
        L.orc_set_counters.argtypes = [vp, u64, u32]
        L.orc_set_trace.restype = C.c_int
        L.orc_set_trace.argtypes = [vp, C.c_int]
        L.orc_get_trace.argtypes = [vp] + [vp] * 7
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


class IndexedOracle:
    """Estimators with global ids [first, first+count) of r (the whole stream's r)."""

    def __init__(self, r: int, seed: int, first: int = 0, count: int | None = None):
        self.r, self.seed, self.first = r, seed, first
        self.count = r - first if count is None else count
        self._h = lib().orc_create(r, seed, first, self.count)
        if not self._h:
            raise ValueError("orc_create failed (r == 0 or bad shard)")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().orc_destroy(h)
            self._h = None

    def push_batch(self, edges) -> int:
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
        return lib().orc_push_batch(self._h, _ptr(e), e.shape[0])

    def push_batch_forced(self, edges, d1, d2) -> int:
        """Test wiring: the batch update with every estimator's Step 1 draw d1[i] (over |W|+|E|) and
        Step 2 draw d2[i] (over chi^- + chi^+, used only when chi^+ > 0) supplied."""
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
        a = np.ascontiguousarray(np.asarray(d1, dtype=np.uint64).reshape(self.count))
        b = np.ascontiguousarray(np.asarray(d2, dtype=np.uint64).reshape(self.count))
        return lib().orc_push_batch_forced(self._h, _ptr(e), e.shape[0], _ptr(a), _ptr(b))

    def set_estimator(self, i, r1, p1, r2, p2, c, closed):
        """Test wiring: overwrite local estimator i (no validation)."""
        a = np.asarray(r1, np.uint32)
        b = np.asarray(r2, np.uint32)
        lib().orc_set_estimator(self._h, int(i), _ptr(a), int(p1), _ptr(b), int(p2), int(c), int(closed))

    def set_counters(self, m, b):
        lib().orc_set_counters(self._h, int(m), int(b))

    def set_trace(self, on: bool = True):
        """Test wiring: record the per-step values of every later batch (trace())."""
        if lib().orc_set_trace(self._h, 1 if on else 0) != 0:
            raise MemoryError("orc_set_trace")

    def trace(self):
        """Per-step values of the last batch: j (Step 1 replacement index, 2^32-1 = retained), chi_m (chi^-),
        ld, rd (ranks; chi^+ = ld + rd), d2 (Step 2 draw, 2^64-1 = none), k2 (batch position of the new f2,
        2^32-1 = kept), closed (after Step 3)."""
        n = self.count
        out = dict(j=np.empty(n, np.uint32), chi_m=np.empty(n, np.uint32), ld=np.empty(n, np.uint32),
                   rd=np.empty(n, np.uint32), d2=np.empty(n, np.uint64), k2=np.empty(n, np.uint32),
                   closed=np.empty(n, np.uint8))
        lib().orc_get_trace(self._h, *[_ptr(out[f]) for f in ("j", "chi_m", "ld", "rd", "d2", "k2", "closed")])
        return out

    def state(self):
        n = self.count
        r1 = np.empty((n, 2), np.uint32)
        r2 = np.empty((n, 2), np.uint32)
        p1 = np.empty(n, np.uint64)
        p2 = np.empty(n, np.uint64)
        c = np.empty(n, np.uint32)
        closed = np.empty(n, np.uint8)
        lib().orc_get_state(self._h, _ptr(r1), _ptr(p1), _ptr(r2), _ptr(p2), _ptr(c), _ptr(closed))
        return dict(r1=r1, p1=p1, r2=r2, p2=p2, c=c, closed=closed)

    def closed_sum(self) -> int:
        return int(lib().orc_closed_sum(self._h))

    def counters(self):
        m, b = C.c_uint64(), C.c_uint32()
        lib().orc_counters(self._h, C.byref(m), C.byref(b))
        return int(m.value), int(b.value)

    def estimate(self) -> float:
        m, _ = self.counters()
        return float(m) * float(self.closed_sum()) / float(self.r)


def philox(ctr, key):
    c = np.asarray(ctr, np.uint32)
    k = np.asarray(key, np.uint32)
    out = np.empty(4, np.uint32)
    lib().orc_philox(_ptr(c), _ptr(k), _ptr(out))
    return tuple(int(v) for v in out)


def threads() -> int:
    return int(lib().orc_threads())
