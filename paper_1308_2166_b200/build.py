"""Builds the sm_100a shared library libtc_b200.so in-tree with nvcc (no torch JIT cache)."""
from __future__ import annotations

import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libtc_b200.so")
SOURCES = ["kernels.cu", "event.cu", "engine.cu", "exact.cu", "ingest.cpp"]
HEADERS = ["kernels.h", "event.h", "index.cuh", "philox.cuh", os.path.join("..", "..", "include", "tc.h")]

NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-pthread", "-shared", "-Xptxas", "-v"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a library")


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(os.path.join(CSRC, f)) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Build the library (out: another path for an experimental variant, e.g. with -D defines)."""
    if out == LIB and not force and not stale():
        return LIB
    out = os.path.abspath(out)
    tmp = out + ".tmp%d" % os.getpid()
    cmd = [nvcc()] + NVCC_FLAGS + [f"-D{d}" for d in defines] + ["-o", tmp] + [os.path.join(CSRC, f) for f in SOURCES]
    res = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    if verbose:
        print(res.stderr)
    if out == LIB:
        with open(os.path.join(CSRC, "ptxas.log"), "w") as f:
            f.write(res.stderr)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force=True, verbose=True))
