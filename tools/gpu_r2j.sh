#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_configs.py > gpurun_out/gpu_rest.log 2>&1; echo "rest rc=$?"; tail -2 gpurun_out/gpu_rest.log
timeout 1200 python -m pytest tests/test_gpu_configs.py -x -q > gpurun_out/cfg.log 2>&1; echo "cfg rc=$?"; tail -2 gpurun_out/cfg.log
for c in C2 C3; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 28 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"; done
TC_LIB_PATH=paper_1308_2166_b200/libtc_pb12.so timeout 600 python bench.py --config C3 --no-cpu-baseline --no-e2e --steps 28 > gpurun_out/bench_C3_pb12.json 2> gpurun_out/bench_C3_pb12.err; echo "C3 pb12 rc=$?"
