#!/bin/bash
# event mode vs bulk: C5 whole-stream passes at small w, C1
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for lw in ${LWS:-12 13 14 16}; do
  w=$((1 << lw))
  timeout 900 python bench.py --config C5 --w $w --mode event --whole-stream --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ed_c5_$lw.json 2> gpurun_out/ed_c5_$lw.err
  echo "event w=2^$lw rc=$?"; tail -2 gpurun_out/ed_c5_$lw.err
done
timeout 600 python bench.py --config C1 --mode event --steps 100 > gpurun_out/ed_c1.json 2> gpurun_out/ed_c1.err; echo "C1 event rc=$?"; tail -2 gpurun_out/ed_c1.err
python tools/tune_summary.py gpurun_out/ed_*.json
