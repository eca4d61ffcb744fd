#!/bin/bash
# long-run A/B of the W-tile L2 policy (evict_first = default vs evict_last), C1 bench + sampling twin
for rep in 1 2; do
for t in 3,2,0,4 3,3,0,4; do
  timeout -s KILL 600 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 0 --correction-tokens 0 --no-backward-bench --tuning $t > gpurun_out/m.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/m.json')); print('$rep tuning=$t c1', round(d['value']/1e6,4), 'sample', round(d['sample_twin']['tokens_per_s']/1e6,4), d['clocks']['sm_mhz'])"
done
done
