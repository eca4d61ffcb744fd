#!/bin/bash
# A/B of the vocab-slice count S_v: small-N latency and C1 throughput per build
mkdir -p gpurun_out
for lib in libtim libtim_s32 libtim_s64; do
  L=$PWD/paper_2605_14220_b200/$lib.so
  echo "== $lib"
  TIM_LIBRARY=$L timeout -s KILL 300 python scripts/small_n.py
  for c in c1 c2; do
  TIM_LIBRARY=$L timeout -s KILL 600 python bench.py --config $c --steps 5 --no-cpu-baseline --e2e-steps 0 --correction-tokens 0 --no-backward-bench --no-sample-bench > gpurun_out/slices_$lib_$c.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/slices_$lib_$c.json')); print('$c', round(d['value']/1e6,4), 'Mtok/s', round(d['roofline']['achieved'],1), 'TF', d['clocks']['sm_mhz'], d['max_abs_dlogp_vs_oracle'] if 'max_abs_dlogp_vs_oracle' in d else '', d['max_abs_dlogp_across_shapes'])"
  done
done
