"""The bounds-checked build (-DTC_CHECKED, index.cuh TC_CHECK): every kernel path of tools/sanitize_run.py
(C1 batches, a hub stream through the hash, hub-peeling, radix-sort and split-partition paths, the small-batch,
split and one-CTA-index passes, graphs, asynchronous errors, a world-1 NCCL rank handle) runs with the device
checking its computed indices; a violation would fail the push with TC_EINTERNAL.  This stands in for
compute-sanitizer, which the GPU pool refuses (profiles/sanitizer_r02_memcheck_refused.log)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)


def test_checked_build_runs_every_path(tmp_path):
    from paper_1308_2166_b200 import build
    lib = build.build(out=str(tmp_path / "libtc_checked.so"), defines=["TC_CHECKED"])
    env = dict(os.environ, TC_LIB_PATH=lib)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=1200)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "sanitize workload ok" in out.stdout
