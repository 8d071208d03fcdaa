#!/bin/bash
# ncu launch list (device time per kernel) of config-2 ADMM runs (scripts/admm_prof.py).
# $1 = launch cap, $2 = cache control (all = cold, none = warm L2 like the real loop)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control ${2:-all} \
  --csv -c ${1:-400} python scripts/admm_prof.py > gpurun_out/admm_ll.csv 2>&1
grep -E "^\"[0-9]" gpurun_out/admm_ll.csv | python3 -c "
import sys,csv
from collections import defaultdict
agg=defaultdict(lambda:[0,0.0])
for r in csv.reader(sys.stdin):
  if len(r)>14:
    k=r[4].split('(')[0][:60]; agg[k][0]+=1; agg[k][1]+=float(r[14])/1e3
for k,(n,t) in sorted(agg.items(), key=lambda kv:-kv[1][1]): print(f'{n:5d} {t/n:9.2f} us avg  {t:10.1f} us total  {k}')
"
