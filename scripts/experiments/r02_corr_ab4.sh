#!/bin/bash
# Round 2: cp.async ring depth 4 (libtim.so) vs 5 / 6 stages, interleaved.
mkdir -p gpurun_out
for rep in 1 2 3; do
for lib in libtim libtim_s5 libtim_s6; do
  echo -n "$rep $lib "; TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so timeout -s KILL 300 python scripts/corr_time.py
done
done
