#!/bin/bash
# DRAM lines and L2 hits of one mid-stream batch's estimator pass (and vertex kernel) at $CFG under an
# application-replay pipeline capture (no cache control), for each knob set in $AB ("" = default)
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
CFG=${CFG:-C3}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_requests_srcunit_tex_op_read.sum
i=0
for ab in "" $AB; do
  T=""; for kv in ${ab//,/ }; do T="$T --tune $kv"; done
  CMD="python bench.py --config $CFG --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-profile-pass $T"
  ncu --replay-mode application --cache-control none --clock-control none --metrics $M \
      -k regex:"k_update|k_vhash|k_pairs" -s 21 -c 3 --csv --log-file gpurun_out/pipe_upd_$i.csv $CMD > gpurun_out/ncu_upd_$i.log 2>&1
  echo "[$ab] rc=$?"
  grep '^"' gpurun_out/pipe_upd_$i.csv | python3 -c "
import csv,sys,collections
r=list(csv.reader(sys.stdin)); h=r[0]; agg=collections.OrderedDict()
for row in r[1:]:
  d=dict(zip(h,row)); k=d['ID']+' '+d['Kernel Name'][:16]; agg.setdefault(k,{})[d['Metric Name']]=float(d['Metric Value'].replace(',',''))
n=1<<22
for k,m in agg.items():
  print('  ',k, 'rd lines/est %.2f'%(m['dram__bytes_read.sum']/n/128), 'wr B/est %.1f'%(m['dram__bytes_write.sum']/n), 'L2 sect/est %.2f'%(m['lts__t_sectors_srcunit_tex_op_read.sum']/n),'req/est %.2f'%(m['lts__t_requests_srcunit_tex_op_read.sum']/n), 'rd hit %.1f'%(100*m['lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum']/max(1,m['lts__t_sectors_srcunit_tex_op_read.sum'])), 'us %.0f'%(m['gpu__time_duration.sum']/1e3))
"
  i=$((i+1))
done
