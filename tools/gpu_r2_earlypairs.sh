#!/bin/bash
# Full GPU suite + smoke on the main library, then an A/B on the same box: k_pairs forked right behind k_count
# (-DTC_EXP_EARLY_PAIRS: it overlaps the scans, the scatter and the split as well as the vertex phase) against the
# default fork behind the whole partition.  Parity subset on the variant first.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
P=$PWD/paper_1308_2166_b200
B="python bench.py --no-e2e --no-cpu-baseline --steps 28 --warmup 3"
TC_LIB_PATH=$P/libtc_earlypairs.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q -k "not C4 and not C5_sweep" > gpurun_out/ep_parity.log 2>&1; echo "variant parity rc=$?"
tail -1 gpurun_out/ep_parity.log
for i in 1 2; do
  $B > gpurun_out/ep_base_c3_$i.json 2>gpurun_out/ep_err.log; echo "base c3 $i rc=$?"
  TC_LIB_PATH=$P/libtc_earlypairs.so $B > gpurun_out/ep_var_c3_$i.json 2>gpurun_out/ep_err.log; echo "var c3 $i rc=$?"
done
$B --config C2 > gpurun_out/ep_base_c2.json 2>gpurun_out/ep_err.log
TC_LIB_PATH=$P/libtc_earlypairs.so $B --config C2 > gpurun_out/ep_var_c2.json 2>gpurun_out/ep_err.log
$B --config C5 --w 1048576 > gpurun_out/ep_base_c5.json 2>gpurun_out/ep_err.log
TC_LIB_PATH=$P/libtc_earlypairs.so $B --config C5 --w 1048576 > gpurun_out/ep_var_c5.json 2>gpurun_out/ep_err.log
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/ep_*_c*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d['ms_per_step'],4), d['value'])
    except Exception as e: print(f, 'ERR', e)
PY
timeout 1500 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/ep_suite.log 2>&1; echo "suite rc=$?" | tee -a gpurun_out/ep_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/ep_smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/ep_suite.log
