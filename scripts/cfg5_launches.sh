#!/bin/bash
# ncu launch list (device time per kernel) of one config-5 batched SR solve
# (64 x 1024^2, frozen guides, scripts/cfg5_repeat.py with 1 run); warm L2 like the real loop.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none \
  --csv python scripts/cfg5_repeat.py 64 1 > gpurun_out/cfg5_ll.csv 2>&1
grep -E "^\"[0-9]" gpurun_out/cfg5_ll.csv | python3 -c "
import sys,csv
from collections import defaultdict
rows=list(csv.reader(sys.stdin))
# metric rows: one per (launch, metric)
agg=defaultdict(lambda:defaultdict(float)); cnt=defaultdict(set)
for r in rows:
  if len(r)>14:
    k=r[4].split('(')[0][:70]; m=r[12]; v=float(r[14].replace(',',''))
    agg[k][m]+=v; cnt[k].add(r[0])
for k,d in sorted(agg.items(), key=lambda kv:-kv[1]['gpu__time_duration.sum']):
  n=len(cnt[k]); t=d['gpu__time_duration.sum']/1e3
  gb=(d['dram__bytes_read.sum']+d['dram__bytes_write.sum'])/1e9
  print(f'{n:5d} {t/n:9.2f} us avg {t:10.1f} us total {gb:8.2f} GB {gb/(t*1e-6)/1e3 if t else 0:6.2f} TB/s  {k}')
"
