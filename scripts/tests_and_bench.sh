#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/t5.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/t5.log
timeout -s KILL 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
cat gpurun_out/bench.json
for t in 3,2,1,2 3,2,1,8 3,2,0,4; do
  timeout -s KILL 300 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 0 --tuning $t > gpurun_out/sweep_$t.json 2>gpurun_out/sweep_$t.err
  python -c "import json,sys; d=json.load(open('gpurun_out/sweep_$t.json')); print('$t', round(d['value']/1e6,4), 'Mtok/s', round(d['roofline']['achieved'],1), 'TF', d['clocks'])"
done
