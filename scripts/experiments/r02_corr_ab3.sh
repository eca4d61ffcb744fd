#!/bin/bash
# Round 2: correction pass 1 with a per-lane cp.async ring (libtim.so) vs the bulk-copy ring
# (libtim_old.so), interleaved; correction parity tests on the new build first.
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_correct_paths.py tests/test_gpu_correct.py tests/test_gpu_sweep.py -m gpu -q -x > gpurun_out/corr_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/corr_tests.log
for rep in 1 2 3; do
for lib in libtim_old libtim; do
  echo -n "$rep $lib "; TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so timeout -s KILL 300 python scripts/corr_time.py
done
done
REPS=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:correct_local -s 3 -c 1 \
   -o gpurun_out/prof_correct_cpasync -f python scripts/correct_only.py > gpurun_out/ncu_corr.log 2>&1; echo ncu_rc=$?
