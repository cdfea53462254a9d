#!/bin/bash
# round-2 final validation: the whole GPU suite, the bench lines (bulk C3 default / C2 / C1, event C5 w=2^12..2^14 and C1)
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build_smoke.log 2>&1; echo "build+smoke rc=$?"
timeout 3600 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/gpu_suite.log 2>&1; echo "suite rc=$?"; tail -22 gpurun_out/gpu_suite.log
timeout 900 python bench.py > gpurun_out/final_c3.json 2> gpurun_out/final_c3.err; echo "C3 rc=$?"
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err; echo "C2 rc=$?"
timeout 600 python bench.py --config C1 --steps 100 > gpurun_out/final_c1.json 2> gpurun_out/final_c1.err; echo "C1 rc=$?"
for lw in 12 13 14; do
  timeout 900 python bench.py --config C5 --w $((1 << lw)) --mode event --whole-stream --warmup 3 --no-e2e > gpurun_out/event_c5_$lw.json 2> gpurun_out/event_c5_$lw.err; echo "event w=2^$lw rc=$?"
done
timeout 600 python bench.py --config C1 --mode event --steps 100 > gpurun_out/event_c1.json 2> gpurun_out/event_c1.err; echo "C1 event rc=$?"
python tools/tune_summary.py gpurun_out/final_c*.json gpurun_out/event_*.json
