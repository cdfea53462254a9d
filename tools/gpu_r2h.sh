#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python -m pytest tests/test_gpu_parity.py -x -q -k "knobs or fuzz or hub" > gpurun_out/par.log 2>&1; echo "par rc=$?"; tail -1 gpurun_out/par.log
python -m pytest tests/test_gpu_configs.py -x -q -k "C3 or (C5 and (22 or 23 or 24))" > gpurun_out/cfg.log 2>&1; echo "cfg rc=$?"; tail -1 gpurun_out/cfg.log
python -m pytest tests/test_checked_build.py tests/test_bench_contract.py -x -q > gpurun_out/chk.log 2>&1; echo "chk rc=$?"; tail -1 gpurun_out/chk.log
python bench.py --config C3 --no-cpu-baseline --no-e2e --steps 28 > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; echo "C3 rc=$?"
