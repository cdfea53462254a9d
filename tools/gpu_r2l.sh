#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python bench.py --config C1 --steps 100 > gpurun_out/final_c1.json 2> gpurun_out/final_c1.err; echo "C1 rc=$?"
timeout 1200 python bench.py --config C4 --steps 8 --warmup 2 > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err; echo "C4 rc=$?"
bash tools/sweep_c5.sh > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?"; tail -30 gpurun_out/sweep.log
