#!/bin/bash
# Round 2: correction pass-1 variants (occupancy / ring depth) vs the previous build, interleaved.
mkdir -p gpurun_out
for rep in 1 2 3; do
for lib in old m5s4 m6s4 m8s4 m6s5; do
  echo -n "$rep $lib "; TIM_LIBRARY=$PWD/paper_2605_14220_b200/libtim_$lib.so timeout -s KILL 300 python scripts/corr_time.py
done
done
REPS=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:correct_local -s 3 -c 1 \
   -o gpurun_out/prof_correct_r02 -f python scripts/correct_only.py > gpurun_out/ncu_corr.log 2>&1; echo ncu_rc=$?
