#!/bin/bash
# interleaved A/B/C of the epilogue TMEM prefetch: libtim_old (none), libtim (sampling twin),
# libtim_pf2 (sampling twin + log-prob forward); C1 forward bench and the sampling twin
timeout -s KILL 900 python -m pytest tests/test_gpu_logprob.py tests/test_gpu_sample.py tests/test_gpu_graph.py -m "gpu and not slow" -q -x 2>&1 | tail -1
TIM_LIBRARY=$PWD/paper_2605_14220_b200/libtim_pf2.so timeout -s KILL 900 python -m pytest tests/test_gpu_logprob.py -m "gpu and not slow" -q -x 2>&1 | tail -1
for rep in 1 2 3; do
for lib in libtim_old libtim libtim_pf2; do
  L=$PWD/paper_2605_14220_b200/$lib.so
  TIM_LIBRARY=$L timeout -s KILL 300 python scripts/sample_only.py | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read().strip()); print('$rep $lib sample', round(d['tokens_per_s']/1e6,4), d['ids_sum'])"
  TIM_LIBRARY=$L timeout -s KILL 600 python bench.py --steps 10 --no-cpu-baseline --e2e-steps 0 --correction-tokens 0 --no-backward-bench --no-sample-bench > gpurun_out/m.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/m.json')); print('$rep $lib c1', round(d['value']/1e6,4), d['clocks']['sm_mhz'])"
done
done
