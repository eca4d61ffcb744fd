#!/bin/bash
# Round 2 (late): persisting-L2 set-aside 0 (all of L2 to normal accesses) vs the driver default
# (24.9 MB here): correction / PPO passes at 2^27 tokens and the C2 step, interleaved x3.
mkdir -p gpurun_out
for r in 1 2 3; do for mb in 0 -1; do
  timeout -s KILL 900 python bench.py --l2-persist-mb $mb --steps 4 --no-extra-configs --no-backward-bench --no-sample-bench --no-cpu-baseline --e2e-steps 0 > gpurun_out/l2z_$mb.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/l2z_$mb.json')); print('$r l2 $mb value', round(d['value']/1e6,4), 'ms/step', round(d['ms_per_step'],1), 'corr', round(d['correction_roofline']['ms'],4), 'ppo', round(d['ppo_roofline']['ms'],4), d['config'].get('l2_persisting_mb'))"
done; done
