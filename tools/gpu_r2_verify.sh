#!/bin/bash
# Round-2 re-entry check: GPU suite, smoke, default bench line (C3).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/v_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/v_gpu_suite.log 2>&1; echo "suite rc=$?" >> gpurun_out/v_gpu_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/v_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/v_smoke.log
timeout 600 python bench.py > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err; echo "bench rc=$?" >> gpurun_out/v_bench.err
