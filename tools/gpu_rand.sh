#!/bin/bash
# DRAM bytes per random read by load flavour (tools/randbench.cu): rates without ncu, bytes with ncu
cd "$GRAFT_REPO_ROOT" || exit 1
./tools/randbench 1073741824 > gpurun_out/rand_rates.txt 2>&1
./tools/randbench 1073741824 32 >> gpurun_out/rand_rates.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum --clock-control none --csv -k regex:k_read ./tools/randbench 1073741824 > gpurun_out/rand_ncu.csv 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum --clock-control none --csv -k regex:k_read ./tools/randbench 1073741824 32 > gpurun_out/rand_ncu32.csv 2>&1
cat gpurun_out/rand_rates.txt
