#!/bin/bash
# Round 2: fused P = 1 correction (warp-balanced zeroing) vs the split launches, interleaved.
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_correct_paths.py tests/test_gpu_correct.py -m gpu -q -x > gpurun_out/corr_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/corr_tests.log
for rep in 1 2 3; do
  echo -n "$rep split "; SPLIT=1 timeout -s KILL 300 python scripts/corr_time.py
  echo -n "$rep fused "; SPLIT=0 timeout -s KILL 300 python scripts/corr_time.py
done
REPS=1 timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/corr_launches_fused.csv python scripts/correct_only.py > /dev/null 2>&1; echo ncu1_rc=$?
