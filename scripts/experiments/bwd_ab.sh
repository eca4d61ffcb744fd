#!/bin/bash
# interleaved A/B of the head backward between two builds
for rep in 1 2 3; do
for lib in libtim_old libtim; do
  TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so timeout -s KILL 300 python scripts/bwd_bench.py | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$rep', '$lib', round(d['ms_backward'],3), 'ms', round(d['ms_grad_kernel_est'],3), 'grad', round(d['ms_forward'],3), 'fwd')"
done
done
