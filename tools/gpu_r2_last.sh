#!/bin/bash
# Last check of round 2 on a fresh box: GPU suite, smoke, the default bench line (C3), the reference arm
# (bounded), and the ncu launch list of the default bench command.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/l_build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/l_suite.log 2>&1; echo "suite rc=$?" | tee -a gpurun_out/l_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/l_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/l_c3.json 2> gpurun_out/l_c3.err; echo "c3 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/l_ref.json 2> gpurun_out/l_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/l_launches_C3.csv \
    python bench.py --no-e2e --no-cpu-baseline --steps 14 --warmup 3 > gpurun_out/l_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/l_suite.log
