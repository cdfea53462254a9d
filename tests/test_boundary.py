"""CPU-side checks of the boundary: the C-ABI library builds for sm_100a, loads, and exports every
symbol include/tc.h declares; the header's declarations and the binding agree.  No compute calls."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "tc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tc_[a-z_]+)\s*\(", src)))


def test_library_builds_and_exports_header_symbols():
    from paper_1308_2166_b200 import _lib, build
    path = build.build()
    L = ctypes.CDLL(path)
    names = _header_functions()
    assert "tc_create" in names and "tc_push_batch" in names and "tc_estimate" in names and "tc_destroy" in names
    for n in names:
        assert hasattr(L, n), f"{n} declared in include/tc.h but not exported"
    assert set(names) == set(_lib.EXPORTS)


def test_sass_is_sm100a():
    import subprocess
    from paper_1308_2166_b200 import build
    path = build.build()
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_when_library_missing(tmp_path):
    from paper_1308_2166_b200 import _lib
    with pytest.raises(ImportError):
        saved = _lib._lib
        _lib._lib = None
        try:
            _lib.load(str(tmp_path / "missing.so"))
        finally:
            _lib._lib = saved


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1308_2166_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle|#include\s*[<\"].*oracle|liboracle", txt, re.M), f


def test_required_estimators_matches_oracle():
    """tc_required_estimators (host-only, no device needed) against the oracle's sizing helper (Theorem
    mdelta-suffices) and its closed form at ln(1/delta) = 1."""
    import math

    from oracle import nbsi
    from paper_1308_2166_b200 import TCError, required_estimators
    from paper_1308_2166_b200 import build as b
    b.build()
    assert required_estimators(0.5, math.exp(-1), 10, 4, 20) == math.ceil(96 / 0.25 * 2.0)
    for eps, delta, m, D, tau in [(0.1, 0.05, 117_185_083, 33_313, 627_584_181), (0.2, 0.01, 1_000, 59, 10_615),
                                  (0.05, 0.1, 1_806_067_135, 5_214, 4_173_724_142)]:
        assert required_estimators(eps, delta, m, D, tau) == nbsi.required_estimators(eps, delta, m, D, tau)
    for bad in [(0.0, 0.5, 1, 1, 1), (0.1, 1.0, 1, 1, 1), (0.1, 0.5, 1, 1, 0)]:
        with pytest.raises(TCError):
            required_estimators(*bad)
