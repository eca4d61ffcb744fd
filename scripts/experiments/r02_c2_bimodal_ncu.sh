#!/bin/bash
# Round 2 (late): 8 consecutive C2 log-prob launches (scripts/c2_steps.py) under one ncu pass of a
# few metrics: does the slow mode go with DRAM traffic / L2 hit rate / clock?
mkdir -p gpurun_out
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,lts__t_sector_hit_rate.pct"
timeout -s KILL 1200 ncu --metrics $M --clock-control none --csv -k regex:logprob_fwd -s 1 -c 8 \
  --log-file gpurun_out/bim.csv python scripts/c2_steps.py 8 > gpurun_out/bim.log 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/bim.csv')))
h=None; d=collections.defaultdict(dict)
for r in rows:
    if r and r[0]=='ID': h=r; continue
    if h and len(r)==len(h):
        x=dict(zip(h,r)); d[x['ID']][x['Metric Name']]=x['Metric Value']
for k,v in d.items():
    print(k, 'ms', round(float(v['gpu__time_duration.sum'])/1e6,1), 'GHz', round(float(v['sm__cycles_elapsed.avg.per_second'])/1e9,3),
          'DRAM TB', round(float(v['dram__bytes_read.sum'])/1e12,3), 'L2 hit', v['lts__t_sector_hit_rate.pct'])
PY
