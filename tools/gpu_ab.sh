#!/bin/bash
# A/B of prebuilt library variants (TC_LIB_PATH) on the default bench workload, phase times only.
set -u
mkdir -p gpurun_out
for lib in "$@"; do
  echo "== $lib"
  TC_LIB_PATH=$PWD/$lib timeout 600 python bench.py --steps ${STEPS:-60} --warmup 3 --no-cpu-baseline --no-e2e ${BARGS:-} > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -5 gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); r=d['roofline']
print('ms/step %.4f' % d['ms_per_step'], {p: round(v['ms_per_step']*1e3,1) for p, v in r['phases'].items()})"
done
