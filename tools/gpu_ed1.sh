#!/bin/bash
# event mode: GPU parity tests (timeouts per file)
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_event.py -q -x --durations=12 > gpurun_out/ed1.log 2>&1; echo ed1=$?
tail -40 gpurun_out/ed1.log
