python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 300 python bench.py --config C1 --steps 30 --warmup 3 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo "bench c1 rc=$?"
CMD="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 1500 ncu --set full --import-source on --clock-control none -k "regex:k_update|k_vhash|k_vhub|k_count|k_scatter|k_pairs|k_scan" -s 36 -c 7 -f -o gpurun_out/prof_r01 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
