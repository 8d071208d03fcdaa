#!/bin/bash
# Per-kernel device times (ncu launch list) of one adaptive denoise + two frozen
# applies at $1^2 (default 8192), k cache off unless $2 == cache.
n=${1:-8192}
extra=--nocache
[ "$2" == "cache" ] && extra=
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  python scripts/prof_dsg.py $n $extra > gpurun_out/ll_$n.csv 2>&1
grep -E "pnp::" gpurun_out/ll_$n.csv | python3 -c "
import sys,csv
rows={}
for r in csv.reader(sys.stdin):
  if len(r)>14: rows.setdefault((int(r[0]), r[4].split('(')[0][:44]), {})[r[12]] = float(r[14])
for (i,k),m in sorted(rows.items()):
  t=m['gpu__time_duration.sum']/1e3
  b=(m['dram__bytes_read.sum']+m['dram__bytes_write.sum'])/1e6
  print(f'{i:3d} {k:44s} {t:9.1f} us  {b:9.1f} MB  {b/t:6.2f} TB/s')
"
