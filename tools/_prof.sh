python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && timeout 1500 ncu --set full --import-source on --clock-control none -k "regex:k_update|k_vhash|k_vhub|k_count|k_scatter|k_pairs" -s 18 -c 6 -f -o gpurun_out/prof19 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
