#!/bin/bash
# A/B the L2-policy / sleep knobs on C1 (results are bit-identical; only speed changes)
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -q -x -k "raw_accumulators or toy_parity or qwen_head or invariance or temperature" > gpurun_out/t3.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/t3.log
for t in 0,0,0 0,0,1 3,1,1 3,2,1 3,0,0 1,2,1; do
  timeout -s KILL 300 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 0 --tuning $t > gpurun_out/sweep_$t.json 2>gpurun_out/sweep_$t.err
  python -c "import json,sys; d=json.load(open('gpurun_out/sweep_$t.json')); print('$t', round(d['value']/1e6,4), 'Mtok/s', round(d['roofline']['achieved'],1), 'TF', d['clocks'])"
done
