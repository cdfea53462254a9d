#!/bin/bash
# per-step DRAM lines of the estimator pass at C3: the split pass (k_u1..k_r) under an application-replay
# pipeline capture (no cache control), one mid-stream batch; the fused k_update of the same batch alongside
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_requests_srcunit_tex_op_read.sum
CMD="python bench.py --config C3 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-profile-pass"
$CMD --tune split_kernels=1 > gpurun_out/split_plain.log 2>&1 || { echo "plain split run failed"; tail gpurun_out/split_plain.log; exit 1; }
ncu --replay-mode application --cache-control none --clock-control none --metrics $M \
    -k regex:"k_u[1-4]|k_r_reduce" -s 35 -c 5 --csv --log-file gpurun_out/pipe_split_C3.csv $CMD --tune split_kernels=1 > gpurun_out/ncu_split.log 2>&1
echo "split rc=$?"
ncu --replay-mode application --cache-control none --clock-control none --metrics $M \
    -k regex:"k_update" -s 7 -c 1 --csv --log-file gpurun_out/pipe_upd_C3.csv $CMD > gpurun_out/ncu_upd.log 2>&1
echo "upd rc=$?"
