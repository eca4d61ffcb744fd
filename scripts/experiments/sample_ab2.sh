#!/bin/bash
# sampling-twin A/B of two builds: sampling tests + digests + interleaved timings (3 reps)
timeout -s KILL 900 python -m pytest tests/test_gpu_sample.py tests/test_gpu_logprob.py -m gpu -q -x 2>&1 | tail -1
for lib in libtim_old libtim; do echo -n "$lib "; TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so timeout -s KILL 300 python scripts/digest.py; done
for rep in 1 2 3; do
for lib in libtim_old libtim; do
  TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so timeout -s KILL 300 python scripts/sample_only.py | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read().strip()); print('$rep $lib sample', round(d['tokens_per_s']/1e6,4), d['ids_sum'])"
done
done
