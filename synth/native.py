"""ctypes front end of synth/gen.c: seeded synthetic streams in seconds (C2-C5 sizes).

Inputs only (no arithmetic of the method); built with gcc (OpenMP) into synth/libsynth.so by
``build()``, which ``__graft_entry__.build()`` also calls.  See gen.c for the recipe.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "gen.c")
LIB = os.path.join(HERE, "libsynth.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-Wall",
                               "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        L.gen_rmat.restype = C.c_int64
        L.gen_rmat.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_void_p]
        L.gen_chung_lu.restype = C.c_int64
        L.gen_chung_lu.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.c_uint64, C.c_void_p]
        L.gen_threads.restype = C.c_int
        _lib = L
    return _lib


def rmat(scale: int, edge_factor: int = 16, seed: int = 1, abcd=(0.57, 0.19, 0.19, 0.05)) -> np.ndarray:
    """R-MAT(a, b, c, d), 2^scale vertex ids, edge_factor * 2^scale draws; simple graph, relabelled,
    random order and orientation -> (m, 2) uint32."""
    nd = edge_factor << scale
    out = np.empty((nd, 2), np.uint32)
    a, b, c, _ = abcd
    k = lib().gen_rmat(int(scale), nd, int(seed), float(a), float(b), float(c), out.ctypes.data_as(C.c_void_p))
    if k < 0:
        raise MemoryError("gen_rmat failed")
    return out[:k]


def chung_lu(n: int, m: int, gamma: float = 2.1, dmax: float = 66626.0, seed: int = 1) -> np.ndarray:
    """Chung-Lu power law with m unique edges -> (m, 2) uint32 (see gen.c)."""
    out = np.empty((m, 2), np.uint32)
    k = lib().gen_chung_lu(int(n), int(m), float(gamma), float(dmax), int(seed), out.ctypes.data_as(C.c_void_p))
    if k < 0:
        raise MemoryError("gen_chung_lu failed")
    return out
