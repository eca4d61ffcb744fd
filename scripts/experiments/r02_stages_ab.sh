#!/bin/bash
# Round 2: forward-kernel SMEM ring depth 6 (libtim.so) vs 7 (libtim_st7.so), sampling twin and C1
# log-prob, interleaved.
mkdir -p gpurun_out
for rep in 1 2 3; do
for lib in libtim libtim_st7; do
  L=$PWD/paper_2605_14220_b200/$lib.so
  echo -n "$rep $lib sample "; REPS=10 TIM_LIBRARY=$L timeout -s KILL 300 python scripts/sample_only.py
  TIM_LIBRARY=$L timeout -s KILL 600 python bench.py --config c1 --steps 10 --no-cpu-baseline --e2e-steps 0 --correction-tokens 0 --no-backward-bench --no-sample-bench --no-extra-configs > gpurun_out/m.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/m.json')); print('$rep $lib c1', round(d['value']/1e6,4), d['clocks']['sm_mhz'])"
done
done
