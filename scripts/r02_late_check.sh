#!/bin/bash
# Round 2 (late session): PPO / correction GPU tests incl. the lock-step edge test, compute-sanitizer
# memcheck / racecheck / synccheck over every kernel (scripts/sanitize.py).
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests/test_gpu_ppo.py tests/test_gpu_correct.py tests/test_gpu_robustness.py -m gpu -q -x > gpurun_out/late_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/late_tests.log
bash scripts/sanitize.sh
