#!/bin/bash
# Interleaved A/B of the d = 4096 schedule knobs on full C2 (thermal drift cancels out)
mkdir -p gpurun_out
for rep in 1 2; do
for t in default 3,1,1,1,4 3,1,1,2,4 3,2,1,2,4; do
  if [ "$t" = default ]; then arg=""; else arg="--tuning $t"; fi
  timeout -s KILL 600 python bench.py --config c2 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --correction-tokens 0 --no-backward-bench --no-sample-bench $arg > gpurun_out/c2ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/c2ab.json')); print('$rep', '$t', round(d['value']/1e6,4), 'Mtok/s', round(d['roofline']['achieved'],1), 'TF', d['clocks']['sm_mhz'])"
done
done
