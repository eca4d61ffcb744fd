#!/bin/bash
# Round 2 (late): bench.py C2 line with the 48 MB persisting-L2 set-aside (default) vs the driver
# default (--l2-persist-mb -1), interleaved x2; the new robustness test first.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_robustness.py -m gpu -q 2>&1 | tail -1
for r in 1 2; do for mb in 48 -1; do
  timeout -s KILL 900 python bench.py --l2-persist-mb $mb --no-extra-configs --no-backward-bench --no-sample-bench --no-cpu-baseline --e2e-steps 2 > gpurun_out/l2_$mb.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/l2_$mb.json')); print('$r l2 $mb value', round(d['value']/1e6,4), 'ms/step', round(d['ms_per_step'],1), 'e2e', round(d['e2e']['value']/1e6,4), 'corr', round(d['correction_roofline']['ms'],4), 'ppo', round(d['ppo_roofline']['ms'],4), d['config'].get('l2_persisting_mb'))"
done; done
