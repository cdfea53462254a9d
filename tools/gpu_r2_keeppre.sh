#!/bin/bash
# A/B on one box: k_vhash / k_vhub keeping each arc's partition position from the first read (-DTC_EXP_KEEPPRE)
# instead of re-reading the arc in phase 4.  Parity subset on the variant, then C3 and C2 lines, interleaved.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
V=$PWD/paper_1308_2166_b200/libtc_keeppre.so
[ -f "$V" ] || exit 1
TC_LIB_PATH=$V timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q -k "not C4 and not C5_sweep" > gpurun_out/kp_parity.log 2>&1; echo "variant parity rc=$?"
tail -2 gpurun_out/kp_parity.log
B="python bench.py --no-e2e --no-cpu-baseline --steps 28 --warmup 3"
for i in 1 2; do
  $B > gpurun_out/kp_base_c3_$i.json 2>gpurun_out/kp_err.log; echo "base c3 $i rc=$?"
  TC_LIB_PATH=$V $B > gpurun_out/kp_var_c3_$i.json 2>gpurun_out/kp_err.log; echo "var c3 $i rc=$?"
done
$B --config C2 > gpurun_out/kp_base_c2.json 2>gpurun_out/kp_err.log
TC_LIB_PATH=$V $B --config C2 > gpurun_out/kp_var_c2.json 2>gpurun_out/kp_err.log
python - <<'P'
import json,glob
for f in sorted(glob.glob('gpurun_out/kp_*_c*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); k=d['roofline']['kernels']
        print(f, round(d['ms_per_step'],4), {n:round(k[n]['ms_per_launch']*1e3,1) for n in ('k_vhash','k_vhub','k_update') if n in k})
    except Exception as e: print(f, 'ERR', e)
P
