#!/bin/bash
# Round 2: full GPU suite on the new build, then the fused P = 1 correction vs the split launches
# vs the previous build (interleaved), and a launch list of one fused tim_correct.
mkdir -p gpurun_out
timeout -s KILL 1800 python -m pytest tests -m gpu -q -x > gpurun_out/tests_gpu.log 2>&1; echo tests_rc=$?; tail -4 gpurun_out/tests_gpu.log
for rep in 1 2 3; do
  echo -n "$rep old   "; TIM_LIBRARY=$PWD/paper_2605_14220_b200/libtim_old.so timeout -s KILL 300 python scripts/corr_time.py
  echo -n "$rep split "; SPLIT=1 timeout -s KILL 300 python scripts/corr_time.py
  echo -n "$rep fused "; SPLIT=0 timeout -s KILL 300 python scripts/corr_time.py
done
REPS=1 timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/corr_launches_fused.csv python scripts/correct_only.py > /dev/null 2>&1; echo ncu1_rc=$?
