#!/bin/bash
# C5 batch-size sweep (R-MAT scale 22, r = 2^22): one bench line per w
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for lw in 12 16 20 22 23 24; do
  w=$((1 << lw)); st=$(( (1 << 26) / w )); [ $st -gt 200 ] && st=200; [ $st -lt 4 ] && st=4
  timeout 900 python bench.py --config C5 --w $w --steps $st --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sweep_$lw.json 2> gpurun_out/sweep_$lw.err
  echo "w=2^$lw rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/sweep_$lw.json')); r=d['roofline']
print('  ms/step %.4f edges/s %.3e' % (d['ms_per_step'], d['value']), {p: round(v['ms_per_step']*1e3,1) for p, v in r['phases'].items()})" 2>/dev/null || tail -3 gpurun_out/sweep_$lw.err
done
