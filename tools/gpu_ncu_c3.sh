#!/bin/bash
# ncu evidence at C3: (1) --set full on the top kernels (kernel replay, cold L2), (2) the pipeline's own DRAM
# bytes and L2 hit rates per kernel (application replay, --cache-control none: every pass reruns the program,
# so each kernel sees the L2 contents its predecessors left)
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
CFG=${CFG:-C3}
CMD="python bench.py --config $CFG --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-profile-pass"
$CMD > gpurun_out/plain_ncu.log 2>&1 || { echo "plain run failed"; exit 1; }
[ "${SKIP_FULL:-0}" = 1 ] || ncu --set full --clock-control none --import-source on -k regex:"k_vhash|k_update|k_pairs|k_count|k_scatter|k_split|k_vhub" \
    -s 10 -c 7 -o gpurun_out/prof_$CFG $CMD > gpurun_out/ncu_full_$CFG.log 2>&1
echo "full rc=$?"
ncu --replay-mode application --cache-control none --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_write.sum \
    -k regex:"k_(count|scan|scatter|split|pairs|vh|vb|update)" -s 10 -c 10 --csv --log-file gpurun_out/pipeline_$CFG.csv $CMD > gpurun_out/ncu_pipe_$CFG.log 2>&1
echo "pipe rc=$?"
