#!/bin/bash
# round 2, first measurement call: build, C3 bench line, its ncu launch list, full-size parity tests
cd "$GRAFT_REPO_ROOT" || exit 1
free -g > gpurun_out/host_mem.txt; nproc >> gpurun_out/host_mem.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
echo "bench rc=$?"
python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
echo "bench c2 rc=$?"
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-profile-pass"
$CMD > gpurun_out/plain_c3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c3.csv $CMD > gpurun_out/ncu_c3.log 2>&1
echo "ncu rc=$?"
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q --durations=30 > gpurun_out/configs.log 2>&1
echo "configs rc=$?"
tail -3 gpurun_out/configs.log
