#!/bin/bash
# Round 2: host-input (e2e) path chunk size, C2 bench, interleaved.
mkdir -p gpurun_out
for rep in 1 2; do
for ch in 65536 262144 524288; do
  TIM_HOST_CHUNK=$ch timeout -s KILL 900 python bench.py --steps 3 --e2e-steps 3 --no-extra-configs --no-backward-bench --no-sample-bench --correction-tokens 0 --no-cpu-baseline > gpurun_out/e2e_$ch.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e2e_$ch.json')); print('$rep chunk $ch value', round(d['value']/1e6,4), 'e2e', round(d['e2e']['value']/1e6,4), d['clocks']['sm_mhz'])"
done
done
