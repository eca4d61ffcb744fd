#!/bin/bash
# Round 2: PPO pass with a per-lane cp.async ring (libtim.so: 128 threads x 4 blocks, 4 stages;
# variants: 5 blocks / 3 stages) vs the register-prefetch kernel (libtim_old.so); PPO parity first.
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_ppo.py tests/test_gpu_robustness.py -m gpu -q -x > gpurun_out/ppo_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/ppo_tests.log
for rep in 1 2 3; do
for lib in libtim_old libtim libtim_pm5 libtim_pst3; do
  echo -n "$rep $lib "; TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so timeout -s KILL 300 python scripts/ppo_only.py $((1<<27)) | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print(round(d['achieved'],1),'GB/s', round(d['ms'],4),'ms')"
done
done
