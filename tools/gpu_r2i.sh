#!/bin/bash
# validation after the k_split restore + the partition-bits experiment; every step under its own timeout
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_configs.py > gpurun_out/gpu_rest.log 2>&1; echo "rest rc=$?"; tail -2 gpurun_out/gpu_rest.log
timeout 600 python bench.py --config C3 --no-cpu-baseline --no-e2e --steps 28 > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; echo "C3 rc=$?"
TC_LIB_PATH=paper_1308_2166_b200/libtc_pb11.so timeout 600 python bench.py --config C3 --no-cpu-baseline --no-e2e --steps 28 > gpurun_out/bench_C3_pb11.json 2> gpurun_out/bench_C3_pb11.err; echo "C3 pb11 rc=$?"
TC_LIB_PATH=paper_1308_2166_b200/libtc_pb11.so timeout 600 python bench.py --config C2 --no-cpu-baseline --no-e2e --steps 28 > gpurun_out/bench_C2_pb11.json 2> gpurun_out/bench_C2_pb11.err; echo "C2 pb11 rc=$?"
