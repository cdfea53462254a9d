#!/bin/bash
# Session-3 evidence for the current kernels: bench lines (C3 default with cpu_baseline + e2e, C2, C1), the ncu
# launch list of the C3 bench command, --set full on the hot kernels (a mid-stream batch), the pipeline capture
# (C3, C2: application replay, no cache control, the 8th batch of the stream)
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python bench.py > gpurun_out/final_c3.json 2> gpurun_out/final_c3.err; echo "C3 rc=$?"
timeout 600 python bench.py --config C2 > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err; echo "C2 rc=$?"
timeout 600 python bench.py --config C1 --steps 100 > gpurun_out/final_c1.json 2> gpurun_out/final_c1.err; echo "C1 rc=$?"
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-profile-pass"
timeout 600 $CMD > gpurun_out/plain_c3.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c3.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
MCMD="python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-profile-pass"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_vhash|k_update|k_pairs|k_split|k_scatter|k_count|k_vhub" \
    -s 49 -c 7 -o gpurun_out/prof_c3 $MCMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
ncu -i gpurun_out/prof_c3.ncu-rep --page raw --csv > gpurun_out/prof_c3_raw.csv 2>/dev/null
for CFG in C3 C2; do
  PCMD="python bench.py --config $CFG --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-profile-pass"
  timeout 1500 ncu --replay-mode application --cache-control none --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum \
    -k regex:"k_(count|scan|scatter|split|pairs|vh|vb|update)" -s 70 -c 10 --csv --log-file gpurun_out/pipeline_$CFG.csv $PCMD > gpurun_out/ncu_pipe_$CFG.log 2>&1
  echo "pipe $CFG rc=$?"
done
