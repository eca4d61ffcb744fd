#!/bin/bash
for rep in 1 2; do
for lib in libtim libtim_s72; do
  L=$PWD/paper_2605_14220_b200/$lib.so
  TIM_LIBRARY=$L timeout -s KILL 300 python scripts/small_n.py | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$rep $lib', d['slices'], d['ms'])"
  TIM_LIBRARY=$L timeout -s KILL 600 python bench.py --steps 10 --no-cpu-baseline --e2e-steps 0 --correction-tokens 0 --no-backward-bench --no-sample-bench > gpurun_out/s.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/s.json')); print('$rep $lib c1', round(d['value']/1e6,4), d['clocks']['sm_mhz'])"
done
done
