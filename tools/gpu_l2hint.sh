#!/bin/bash
# tools/l2hint.cu: rates, then DRAM bytes and L2 hits per kernel under ncu
cd "$GRAFT_REPO_ROOT" || exit 1
for mb in 32 48 64; do ./tools/l2hint $((mb << 20)); done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none --cache-control none --csv -k k_mix ./tools/l2hint $((48 << 20)) > gpurun_out/l2hint.csv 2>&1
grep '^"' gpurun_out/l2hint.csv | python3 -c "
import csv,sys,collections
r=list(csv.reader(sys.stdin)); h=r[0]; agg=collections.OrderedDict()
for row in r[1:]:
  d=dict(zip(h,row)); agg.setdefault(d['ID']+' '+d['Kernel Name'][:16],{})[d['Metric Name']]=float(d['Metric Value'].replace(',',''))
for k,m in agg.items(): print(k, 'dramB/pair %.1f'%(m['dram__bytes_read.sum']/(1<<25)), 'hit %.1f'%(100*m['lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum']/m['lts__t_sectors_srcunit_tex_op_read.sum']), 'us %.0f'%(m['gpu__time_duration.sum']/1e3))
"
