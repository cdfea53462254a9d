"""bench.py's reference arm (the CPU oracle, runnable here) prints one JSON line with the contract's keys."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["config"]["workload"].startswith("C1")


import pytest  # noqa: E402


@pytest.mark.gpu
def test_b200_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "C1", "--steps", "6",
                          "--warmup", "3", "--no-cpu-baseline"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "e2e", "gpu_launches"):
        assert k in d, k
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic", "kernel", "kernels", "whole_step"):
        assert k in r, k
    assert 0 < r["frac"] < 1 and d["gpu_launches"] >= 6 * 3 and d["value"] > 0  # C1: desc + small index + update
    # the dominant kernel is the one with the largest measured time, and the shares add up
    ks = r["kernels"]
    assert r["kernel"] == max(ks, key=lambda k: ks[k]["ms_per_launch"] * ks[k]["launches"])
    assert abs(sum(v["share_of_kernel_time"] for v in ks.values()) - 1) < 1e-6
    assert 0 < r["whole_step"]["frac"] < 1
    assert d["cpu_baseline"]["cpu_model"] if "cpu_baseline" in d else True
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d.get("e2e_results_match_tc_estimate") is True


@pytest.mark.gpu
def test_b200_arm_event_mode_json_line():
    """--mode event: the same contract, the event kernels attributed, the event oracle as cpu_baseline."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "C1", "--mode", "event",
                          "--whole-stream", "--warmup", "3"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["config"]["mode"] == "event" and d["steps"] == d["config"]["batches_per_stream"]
    ks = d["roofline"]["kernels"]
    assert {"k_ed_front", "k_ed_process"} <= set(ks) and "k_update" not in ks
    assert d["roofline"]["events_per_batch"]["visited"] > 0
    assert "oracle/ed.c" in d["cpu_baseline"]["sample"] and d["value"] > 0
    assert d.get("e2e_results_match_tc_estimate") is True
