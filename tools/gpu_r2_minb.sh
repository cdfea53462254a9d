#!/bin/bash
# A/B on one box: k_update at 3 and 2 CTAs/SM (80 / 110 registers, no spills) against the default 4 (64 registers,
# 80-100 B of spills); the main library now keeps each arc's partition position in k_vhash / k_vhub (parity subset).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_event.py -m gpu -x -q -k "not C4 and not C5_sweep" > gpurun_out/mb_parity.log 2>&1; echo "main parity rc=$?"
tail -2 gpurun_out/mb_parity.log
B="python bench.py --no-e2e --no-cpu-baseline --steps 28 --warmup 3"
P=$PWD/paper_1308_2166_b200
for i in 1 2; do
  $B > gpurun_out/mb_base_c3_$i.json 2>gpurun_out/mb_err.log; echo "base c3 $i rc=$?"
  for m in 3 2; do
    TC_LIB_PATH=$P/libtc_minb$m.so $B > gpurun_out/mb_m${m}_c3_$i.json 2>gpurun_out/mb_err.log; echo "minb$m c3 $i rc=$?"
  done
done
for m in 3 2; do TC_LIB_PATH=$P/libtc_minb$m.so $B --config C2 > gpurun_out/mb_m${m}_c2.json 2>gpurun_out/mb_err.log; done
$B --config C2 > gpurun_out/mb_base_c2.json 2>gpurun_out/mb_err.log
python - <<'P'
import json,glob
for f in sorted(glob.glob('gpurun_out/mb_*_c*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); k=d['roofline']['kernels']
        print(f, round(d['ms_per_step'],4), {n:round(k[n]['ms_per_launch']*1e3,1) for n in ('k_vhash','k_vhub','k_update') if n in k})
    except Exception as e: print(f, 'ERR', e)
P
