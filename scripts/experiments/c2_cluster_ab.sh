#!/bin/bash
# full C2: default (clusters of one CTA pair) vs 2-pair clusters sharing W tiles by TMA multicast
for rep in 1 2; do
for cp in 0 2; do
  if [ "$cp" = 0 ]; then arg=""; else arg="--cluster-pairs $cp"; fi
  timeout -s KILL 600 python bench.py --config c2 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --correction-tokens 0 --no-backward-bench --no-sample-bench $arg > gpurun_out/c2c.json 2>gpurun_out/c2c.err
  python -c "import json; d=json.load(open('gpurun_out/c2c.json')); print('$rep', 'cluster_pairs=$cp', round(d['value']/1e6,4), 'Mtok/s', round(d['roofline']['achieved'],1), 'TF', d['clocks']['sm_mhz'], d['max_abs_dlogp_across_shapes'])" || tail -3 gpurun_out/c2c.err
done
done
