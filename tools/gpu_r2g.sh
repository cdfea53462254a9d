#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_configs.py > gpurun_out/gpu_rest.log 2>&1; echo "rest rc=$?"; tail -2 gpurun_out/gpu_rest.log
for c in C1 C2 C3; do python bench.py --config $c --no-cpu-baseline --no-e2e --steps 28 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"; done
python bench.py --config C5 --w 4096 --steps 64 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_4096.json 2> gpurun_out/bench_c5_4096.err; echo "c5 rc=$?"
