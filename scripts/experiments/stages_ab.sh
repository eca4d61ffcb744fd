#!/bin/bash
# Interleaved A/B of the forward kernel's SMEM pipeline depth on C1
mkdir -p gpurun_out
for rep in 1 2; do
for lib in libtim libtim_st5 libtim_st7; do
  TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so timeout -s KILL 600 python bench.py --steps 10 --e2e-steps 0 --no-cpu-baseline --correction-tokens 0 --no-backward-bench --no-sample-bench > gpurun_out/st.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/st.json')); print('$rep', '$lib', round(d['value']/1e6,4), 'Mtok/s', round(d['roofline']['achieved'],1), 'TF', d['clocks']['sm_mhz'])"
done
done
