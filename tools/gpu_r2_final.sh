#!/bin/bash
# End of round 2: the GPU suite and the bench lines touched by the small-index default (C1, C5 w=2^12 bulk and
# event, event C1), plus the default C3 line.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/f_suite.log 2>&1; echo "suite rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --config C1 --steps 100 > gpurun_out/f_c1.json 2> gpurun_out/f_c1.err; echo "c1 rc=$?"
timeout 600 python bench.py --config C1 --steps 100 --mode event > gpurun_out/f_ev_c1.json 2> gpurun_out/f_ev_c1.err; echo "ev c1 rc=$?"
timeout 900 python bench.py --config C5 --w 4096 --mode event --whole-stream > gpurun_out/f_ev_c5_12.json 2> gpurun_out/f_ev_c5_12.err; echo "ev c5 rc=$?"
timeout 600 python bench.py --config C5 --w 4096 --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/f_c5_12.json 2> gpurun_out/f_c5_12.err; echo "c5 12 rc=$?"
timeout 900 python bench.py > gpurun_out/f_c3.json 2> gpurun_out/f_c3.err; echo "c3 rc=$?"
