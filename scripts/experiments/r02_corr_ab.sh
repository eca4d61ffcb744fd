#!/bin/bash
# Round 2: correction / PPO kernel rework -- parity tests on the new build, then interleaved
# 2^27-token timings of libtim_old.so (previous build) vs libtim.so.
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_correct_paths.py tests/test_gpu_correct.py tests/test_gpu_sweep.py tests/test_gpu_ppo.py -m gpu -q -x > gpurun_out/corr_tests.log 2>&1; echo tests_rc=$?; tail -15 gpurun_out/corr_tests.log
for rep in 1 2 3; do
for lib in libtim_old libtim; do
  L=$PWD/paper_2605_14220_b200/$lib.so
  TIM_LIBRARY=$L timeout -s KILL 300 python scripts/correct_only.py $((1<<27)) | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('$rep $lib corr', round(d['achieved'],1),'GB/s', round(d['ms'],4),'ms')"
  TIM_LIBRARY=$L timeout -s KILL 300 python scripts/ppo_only.py $((1<<27)) | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('$rep $lib ppo', round(d['achieved'],1),'GB/s', round(d['ms'],4),'ms')"
done
done
REPS=1 timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second --clock-control none --csv \
   --log-file gpurun_out/corr_launches.csv python scripts/correct_only.py > /dev/null 2>&1; echo ncu1_rc=$?
