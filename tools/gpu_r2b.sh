#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python -m pytest tests/test_gpu_nccl.py tests/test_gpu_api.py -x -q > gpurun_out/nccl.log 2>&1; echo "nccl rc=$?"; tail -3 gpurun_out/nccl.log
python -m pytest tests/test_gpu_configs.py -x -q -k "full_range or C4" --durations=5 > gpurun_out/cfg2.log 2>&1; echo "cfg2 rc=$?"; tail -3 gpurun_out/cfg2.log
python bench.py --no-cpu-baseline > gpurun_out/bench_c3b.json 2> gpurun_out/bench_c3b.err; echo "bench rc=$?"
python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_configs.py > gpurun_out/gpu_rest.log 2>&1; echo "rest rc=$?"; tail -3 gpurun_out/gpu_rest.log
