#!/bin/bash
# Round 2 (late): PPO pass with the branch-free histogram slot (saturating floor-convert + integer
# clamp, per-lane sink slots for A = 0) and the single-product clip (libtim.so) vs the previous
# build (libtim_old.so); later: per-lane slow decision + precomputed sequence limit (libtim) vs v3;
# PPO parity first, then interleaved timing at 2^27 tokens.
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_ppo.py tests/test_gpu_robustness.py -m gpu -q -x > gpurun_out/ppo_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/ppo_tests.log
for rep in 1 2 3; do
for lib in libtim_v3 libtim; do
  echo -n "$rep $lib "; TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so timeout -s KILL 300 python scripts/ppo_only.py $((1<<27)) | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print(round(d['achieved'],1),'GB/s', round(d['ms'],4),'ms')"
done
done
REPS=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:ppo_local -s 3 -c 1 \
   -o gpurun_out/prof_ppo -f python scripts/ppo_only.py > gpurun_out/ncu_full_ppo.log 2>&1; echo ncu_rc=$?
