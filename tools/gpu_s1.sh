#!/bin/bash
# session check: build + smoke, the GPU suite, the default (C3) bench line
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build_smoke.log 2>&1; echo "build+smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/gpu_suite.log 2>&1; echo "suite rc=$?"; tail -22 gpurun_out/gpu_suite.log
timeout 900 python bench.py > gpurun_out/s1_c3.json 2> gpurun_out/s1_c3.err; echo "C3 rc=$?"; cat gpurun_out/s1_c3.json | head -c 600
