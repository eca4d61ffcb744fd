#!/bin/bash
# Round 2: sampling twin with the Gumbel-max pass on a second set of epilogue warps (libtim.so)
# vs one set of epilogue warps running both passes (libtim_ss0.so), interleaved; sampling tests.
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_sample.py -m gpu -q -x > gpurun_out/sample_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/sample_tests.log
for rep in 1 2 3; do
for lib in libtim_ss0 libtim; do
  echo -n "$rep $lib "; REPS=10 TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so timeout -s KILL 300 python scripts/sample_only.py
done
done
REPS=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:logprob_fwd -s 2 -c 1 \
   -o gpurun_out/prof_sample_r02 -f python scripts/sample_only.py > gpurun_out/ncu_sample.log 2>&1; echo ncu_rc=$?
