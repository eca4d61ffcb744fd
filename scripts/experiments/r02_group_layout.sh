#!/bin/bash
# Round 2: C2-shaped (d = 4096) DRAM traffic / L2 hit rate vs which CTA pairs share an M-tile:
# consecutive cluster ids (libtim.so) or ids q and q + ngrp (libtim_gl1.so); then full-C2 timing.
mkdir -p gpurun_out
export PYTHONPATH=$PWD
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,lts__t_sector_hit_rate.pct"
for lib in libtim libtim_gl1; do
  TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so timeout -s KILL 600 ncu --metrics $M --clock-control none --csv -k regex:logprob_fwd -c 2 \
   --log-file gpurun_out/gl_$lib.csv python scripts/c2_diag.py 524288 default 2 > gpurun_out/gl_$lib.txt 2>&1
  echo "== $lib"; python - <<PY
import csv
rows=list(csv.reader(open('gpurun_out/gl_$lib.csv')))
h=None
for r in rows:
    if r and r[0]=='ID': h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r)); print(d['ID'], d['Metric Name'], d['Metric Value'], d['Metric Unit'])
PY
done
for rep in 1 2; do
for lib in libtim libtim_gl1; do
  echo -n "$rep $lib "; TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so timeout -s KILL 600 python scripts/c2_diag.py 2097152 default 3 | tail -1
done
done
