#!/bin/bash
# Round 2 (late): C2 DRAM bytes per log-prob launch, the bench's own launches vs scripts/c2_diag.py, one
# ncu pass of three metrics (no replay-set effects), plus the die map of this box.
mkdir -p gpurun_out
export PYTHONPATH=$PWD
python scripts/die_map_print.py
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum"
timeout -s KILL 900 ncu --metrics $M --clock-control none --csv -k regex:logprob_fwd -s 1 -c 2 \
  --log-file gpurun_out/dram_diag.csv python scripts/c2_diag.py 2097152 default 3 > gpurun_out/dram_diag.log 2>&1
timeout -s KILL 900 ncu --metrics $M --clock-control none --csv -k regex:logprob_fwd -s 2 -c 2 \
  --log-file gpurun_out/dram_bench.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
  --no-extra-configs --no-backward-bench --no-sample-bench --correction-tokens 0 > gpurun_out/dram_bench.log 2>&1
for f in dram_diag dram_bench; do echo "== $f"; python - <<PY
import csv
rows=list(csv.reader(open('gpurun_out/$f.csv')))
h=None
for r in rows:
    if r and r[0]=='ID': h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r)); print(d['ID'], d['Metric Name'], d['Metric Value'], d['Metric Unit'])
PY
done
