#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_event.py -q -x > gpurun_out/si.log 2>&1; echo tests=$?; tail -3 gpurun_out/si.log
timeout 600 python bench.py --config C1 --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/si_c1.json 2>/dev/null; echo c1=$?
timeout 600 python bench.py --config C5 --w 4096 --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/si_c5.json 2>/dev/null; echo c5=$?
python tools/tune_summary.py gpurun_out/si_*.json
PYTHONPATH=. timeout 300 python tools/dbg/ed_perbatch.py 4096 8000 1000 | head -2
