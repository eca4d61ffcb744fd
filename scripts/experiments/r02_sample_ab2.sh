#!/bin/bash
# Round 2: sampling twin with the max-tree Gumbel chunk (libtim.so) vs the per-column compare /
# select chain (libtim_old.so): identical ids / log-probs required, interleaved timing, C1 batch.
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_sample.py tests/test_gpu_schedule.py -m gpu -q -x > gpurun_out/sample_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/sample_tests.log
for rep in 1 2 3; do
for lib in libtim_old libtim; do
  echo -n "$rep $lib "; REPS=10 TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so timeout -s KILL 300 python scripts/sample_only.py
done
done
