#!/bin/bash
# long-run A/B of sleeping vs spinning mbarrier waits on C2 (d = 4096) and the head backward
for rep in 1 2; do
for t in 3,2,1,4 3,2,0,4; do
  timeout -s KILL 900 python bench.py --config c2 --steps 4 --no-cpu-baseline --e2e-steps 0 --correction-tokens 0 --no-sample-bench --tuning $t > gpurun_out/m.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/m.json')); print('$rep tuning=$t c2', round(d['value']/1e6,4), 'bwd', round(d['head_backward']['tokens_per_s']/1e6,4), 'saved', round(d['head_backward']['saved']['tokens_per_s']/1e6,4), d['clocks']['sm_mhz'])"
done
done
