#!/bin/bash
# One gpurun call: build, GPU parity tests, a bench line, then ONE `ncu --set full` capture of the hot
# kernels of a short bench run (only after that same command exited 0 without ncu).
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
if [ "${TESTS:-1}" = 1 ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
fi
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
CMD="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain.log 2>&1; rc=$?; echo "plain rc=$rc"
if [ $rc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > /dev/null 2>&1; echo "ncu-list rc=$?"
  timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-k_update|k_vbuckets|k_scatter|k_pbuckets|k_count}" \
      -s ${SKIP:-20} -c ${COUNT:-5} -f -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"
fi
