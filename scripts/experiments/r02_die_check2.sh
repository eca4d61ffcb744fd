#!/bin/bash
# Round 2: die-map probe stability (3 fresh processes) and the DRAM traffic of the bench's own C2
# launches under ncu metrics (die groups on / off).
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for i in 1 2 3; do python scripts/die_map_print.py; done
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum"
for g in 1 0; do
  DIEG=$g timeout -s KILL 900 ncu --metrics $M --clock-control none --csv -k regex:logprob_fwd -s 1 -c 2 \
   --log-file gpurun_out/bb_$g.csv python scripts/c2_diag.py 2097152 default 3 > /dev/null 2>&1
  echo "== DIEG=$g"; python - <<PY
import csv
rows=list(csv.reader(open('gpurun_out/bb_$g.csv')))
h=None
for r in rows:
    if r and r[0]=='ID': h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r)); print(d['ID'], d['Metric Name'], d['Metric Value'], d['Metric Unit'])
PY
done
timeout -s KILL 900 python bench.py --steps 3 --no-extra-configs --no-backward-bench --no-sample-bench --no-cpu-baseline --correction-tokens 0 > gpurun_out/bdm.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bdm.json')); print(d['value'], d['clocks'])"
