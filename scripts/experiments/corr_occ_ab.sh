#!/bin/bash
# correction pass occupancy A/B: blocks per SM (TIM_CORR_MINB) x ring depth (TIM_CORR_STAGES), 2^27 tokens
for lib in libtim_m6s3 libtim_m5s3 libtim_m6s2; do
  TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so timeout -s KILL 900 python -m pytest tests/test_gpu_correct.py -m gpu -q -x 2>&1 | tail -1
done
for rep in 1 2; do
for lib in libtim libtim_m6s3 libtim_m5s3 libtim_m6s2; do
  TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so timeout -s KILL 300 python scripts/correct_only.py $((1<<27)) | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('$rep $lib', round(d['achieved'],1),'GB/s', round(d['ms'],4),'ms')"
done
done
