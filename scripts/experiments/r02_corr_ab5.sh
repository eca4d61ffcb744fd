#!/bin/bash
# Round 2: decisions + stats + zeroing in one launch after pass 1 (libtim.so) vs finish + zero
# launches (libtim_old.so); correction parity tests on the new build first.
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_correct_paths.py tests/test_gpu_correct.py tests/test_gpu_sweep.py tests/test_dist_nccl.py -m gpu -q -x > gpurun_out/corr_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/corr_tests.log
for rep in 1 2 3; do
for lib in libtim_old libtim; do
  echo -n "$rep $lib "; TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so timeout -s KILL 300 python scripts/corr_time.py
done
done
REPS=1 timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/corr_launches_dz.csv python scripts/correct_only.py > /dev/null 2>&1; echo ncu1_rc=$?
