#!/bin/bash
# Round 2: die-aware pair order in the backward GEMMs: tests, then interleaved timing at d = 4096 / 2048.
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout -s KILL 900 python -m pytest tests/test_gpu_schedule.py tests/test_gpu_backward.py -m gpu -q -x > gpurun_out/bwd_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/bwd_tests.log
timeout -s KILL 600 python scripts/experiments/bwd_die_ab.py 4096
timeout -s KILL 600 python scripts/experiments/bwd_die_ab.py 2048
