#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_configs.py > gpurun_out/gpu_rest.log 2>&1; echo "rest rc=$?"; tail -2 gpurun_out/gpu_rest.log
timeout 600 python bench.py --config C1 --steps 100 --no-cpu-baseline > gpurun_out/bench_C1.json 2> gpurun_out/bench_C1.err; echo "C1 rc=$?"
for w in 2048 4096; do timeout 600 python bench.py --config C5 --w $w --steps 64 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_$w.json 2> gpurun_out/bench_c5_$w.err; echo "c5 $w rc=$?"; done
