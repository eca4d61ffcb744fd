#!/bin/bash
# Round 2: is the die-aware grouping active under ncu on the full C2 batch?  die map, then ncu
# metrics of full-C2 launches with the grouping on and off.
mkdir -p gpurun_out
export PYTHONPATH=$PWD
python scripts/die_map_print.py
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,lts__t_sector_hit_rate.pct"
for g in 1 0 1; do
  DIEG=$g timeout -s KILL 900 ncu --metrics $M --clock-control none --csv -k regex:logprob_fwd -c 2 \
   --log-file gpurun_out/dc_$g.csv python scripts/c2_diag.py 2097152 default 2 > /dev/null 2>&1
  echo "== DIEG=$g"; python - <<PY
import csv
rows=list(csv.reader(open('gpurun_out/dc_$g.csv')))
h=None
for r in rows:
    if r and r[0]=='ID': h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r)); print(d['ID'], d['Metric Name'], d['Metric Value'], d['Metric Unit'])
PY
done
