#!/bin/bash
# event-mode whole-stream bench lines (C5 w = 2^12 .. 2^14, C1)
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for lw in 12 13 14; do
  timeout 900 python bench.py --config C5 --w $((1 << lw)) --mode event --whole-stream --warmup 3 --no-e2e > gpurun_out/event_c5_$lw.json 2> gpurun_out/event_c5_$lw.err; echo "event w=2^$lw rc=$?"
done
timeout 600 python bench.py --config C1 --mode event --steps 100 > gpurun_out/event_c1.json 2> gpurun_out/event_c1.err; echo "C1 event rc=$?"
python tools/tune_summary.py gpurun_out/event_*.json
