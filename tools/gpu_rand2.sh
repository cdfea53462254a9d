#!/bin/bash
# L2 residency of a randomly probed table by size (tools/randbench.cu, default-flavour 16-byte reads)
cd "$GRAFT_REPO_ROOT" || exit 1
for mb in 16 32 48 64 96 128; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none --cache-control none --csv -k k_read -c 2 ./tools/randbench $((mb << 20)) > gpurun_out/rand2_$mb.csv 2>&1
  grep '^"' gpurun_out/rand2_$mb.csv | python3 -c "
import csv,sys,collections
r=list(csv.reader(sys.stdin)); h=r[0]; agg=collections.OrderedDict()
for row in r[1:]:
  d=dict(zip(h,row)); agg.setdefault(d['ID'],{})[d['Metric Name']]=float(d['Metric Value'].replace(',',''))
for k,m in agg.items(): print('$mb MB', k, 'dramB/acc %.1f'%(m['dram__bytes_read.sum']/(1<<24)), 'hit %.1f'%(100*m['lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum']/m['lts__t_sectors_srcunit_tex_op_read.sum']), 'us %.0f'%(m['gpu__time_duration.sum']/1e3))
"
done
