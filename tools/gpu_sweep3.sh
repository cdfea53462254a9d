#!/bin/bash
# refresh: the C5 sweep (all w) and the C4 line (pinned-host feed) with the current kernels
cd "$GRAFT_REPO_ROOT" || exit 1
bash tools/sweep_c5.sh > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?"; tail -16 gpurun_out/sweep.log
timeout 1500 python bench.py --config C4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err; echo "C4 rc=$?"
