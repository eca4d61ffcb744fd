#!/bin/bash
# Correction/PPO kernel iteration: parity tests, standalone timing at 2^27 tokens, one ncu capture.
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_correct.py tests/test_gpu_sweep.py tests/test_gpu_ppo.py -m gpu -q -x > gpurun_out/corr_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/corr_tests.log
for i in 1 2; do timeout -s KILL 300 python scripts/correct_only.py $((1<<27)); done
timeout -s KILL 300 python scripts/ppo_only.py $((1<<27)) 2>/dev/null | tail -1
REPS=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:correct_local -s 3 -c 1 \
   -o gpurun_out/prof_correct -f python scripts/correct_only.py > gpurun_out/ncu_corr.log 2>&1; echo ncu_rc=$?
