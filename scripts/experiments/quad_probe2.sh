#!/bin/bash
for t in 3,2,1,0 3,2,1,4 3,2,0,0 3,1,0,8; do
  timeout -s KILL 300 python bench.py --steps 5 --no-cpu-baseline --e2e-steps 0 --correction-tokens 0 --no-sample-bench --cluster-pairs 2 --tuning $t > gpurun_out/q2_$t.json 2>gpurun_out/q2_$t.err
  python -c "import json; d=json.load(open('gpurun_out/q2_$t.json')); print('quad tuning=$t', round(d['value']/1e6,4), 'Mtok/s', round(d['roofline']['achieved'],1), 'TF', d['clocks'])"
done
