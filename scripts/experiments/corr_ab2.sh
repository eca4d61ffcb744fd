#!/bin/bash
# interleaved A/B of the correction kernel between two builds (2^27 tokens)
timeout -s KILL 600 python -m pytest tests/test_gpu_correct.py tests/test_gpu_sweep.py -m gpu -q -x 2>&1 | tail -1
for rep in 1 2 3; do
for lib in libtim_old libtim; do
  TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so timeout -s KILL 300 python scripts/correct_only.py $((1<<27)) | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('$rep $lib', round(d['achieved'],1),'GB/s', round(d['ms'],4),'ms')"
done
done
