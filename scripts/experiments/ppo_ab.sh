#!/bin/bash
# PPO / correction iteration: parity tests, 2^27-token timings, launch lists, one ncu capture of ppo_local.
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_correct.py tests/test_gpu_sweep.py tests/test_gpu_ppo.py -m gpu -q -x > gpurun_out/ppo_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/ppo_tests.log
for i in 1 2; do timeout -s KILL 300 python scripts/ppo_only.py $((1<<27)) | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read().strip().splitlines()[-1]); print('ppo', round(d['achieved'],1),'GB/s', round(d['ms'],4),'ms')"; done
for i in 1 2; do timeout -s KILL 300 python scripts/correct_only.py $((1<<27)) | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('corr', round(d['achieved'],1),'GB/s', round(d['ms'],4),'ms')"; done
REPS=1 timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/ppo_launches.csv python scripts/ppo_only.py > /dev/null 2>&1; echo ncu1_rc=$?
REPS=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:ppo_local -s 3 -c 1 \
   -o gpurun_out/prof_ppo -f python scripts/ppo_only.py > gpurun_out/ncu_ppo.log 2>&1; echo ncu_rc=$?
