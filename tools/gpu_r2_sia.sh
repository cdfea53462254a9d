#!/bin/bash
# k_small_index CTA count (TC_TUNE_SMALL_INDEX_ARCS) at C5 w=2^12 (event mode over the whole stream, bulk) and C1.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "knobs or every_batch_random" > gpurun_out/sia_tests.log 2>&1; echo "tests rc=$?"
for a in 512 256 128 64; do
  timeout 600 python bench.py --config C5 --w 4096 --mode event --whole-stream --no-cpu-baseline --no-e2e --tune small_index_arcs=$a > gpurun_out/sia_ev_$a.json 2>gpurun_out/sia_ev_$a.err; echo "ev $a rc=$?"
  timeout 600 python bench.py --config C5 --w 4096 --steps 200 --no-cpu-baseline --no-e2e --tune small_index_arcs=$a > gpurun_out/sia_bulk_$a.json 2>gpurun_out/sia_bulk_$a.err; echo "bulk $a rc=$?"
  timeout 600 python bench.py --config C1 --steps 100 --no-cpu-baseline --no-e2e --tune small_index_arcs=$a > gpurun_out/sia_c1_$a.json 2>gpurun_out/sia_c1_$a.err; echo "c1 $a rc=$?"
done
