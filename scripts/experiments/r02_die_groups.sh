#!/bin/bash
# Round 2: die-aware M-tile groups (DIEG=1, default) vs cluster-id order (DIEG=0) at d = 4096:
# schedule tests, the probed die map, ncu DRAM / L2 / clock on a 524,288-token call, full-C2 timing.
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout -s KILL 900 python -m pytest tests/test_gpu_schedule.py tests/test_gpu_logprob.py tests/test_gpu_sample.py tests/test_gpu_backward.py -m gpu -q -x > gpurun_out/sched_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/sched_tests.log
python -c "
from paper_2605_14220_b200 import tim
st, die = tim.debug_die_map(); print('die map state', st, 'die-1 SMs', sum(die), ''.join(map(str, die[:148])))"
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,lts__t_sector_hit_rate.pct"
for g in 0 1; do
  DIEG=$g timeout -s KILL 600 ncu --metrics $M --clock-control none --csv -k regex:logprob_fwd -c 2 \
   --log-file gpurun_out/dg_$g.csv python scripts/c2_diag.py 524288 default 2 > gpurun_out/dg_$g.txt 2>&1
  echo "== DIEG=$g"; python - <<PY
import csv
rows=list(csv.reader(open('gpurun_out/dg_$g.csv')))
h=None
for r in rows:
    if r and r[0]=='ID': h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r)); print(d['ID'], d['Metric Name'], d['Metric Value'], d['Metric Unit'])
PY
done
for rep in 1 2 3; do
for g in 0 1; do
  echo -n "$rep DIEG=$g "; DIEG=$g timeout -s KILL 600 python scripts/c2_diag.py 2097152 default 3 | tail -1
done
done
