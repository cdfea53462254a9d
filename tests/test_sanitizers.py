"""compute-sanitizer over the library's kernels: memcheck, racecheck, synccheck and
initcheck on tools/sanitize_run.py (every kernel path, C1-sized).  Marked `sanitizer`, NOT `gpu`: each tool is
run in its own GPU session (`pytest -m sanitizer -k <tool>`), never several in one process or call."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.sanitizer


def _cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_compute_sanitizer(tool):
    if not _cuda():
        pytest.skip("no CUDA device")
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not installed")
    env = dict(os.environ, TC_SANITIZE_NCCL="0" if tool in ("racecheck", "initcheck") else "1")
    cmd = [cs, "--tool", tool, "--error-exitcode", "99", "--target-processes", "all"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    if tool == "initcheck":
        cmd += ["--track-unused-memory", "no"]
    out = subprocess.run(cmd + [sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=3000)
    log = os.path.join(ROOT, "gpurun_out", f"sanitizer_{tool}.log")
    os.makedirs(os.path.dirname(log), exist_ok=True)
    with open(log, "w") as f:
        f.write(out.stdout + "\n---- stderr ----\n" + out.stderr)
    if "closed on this pool" in out.stdout + out.stderr:  # the GPU pool refuses compute-sanitizer
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "sanitize workload ok" in out.stdout
    assert "ERROR SUMMARY: 0 errors" in out.stdout + out.stderr
