#!/bin/bash
# Round 2 (late): PPO pass with the int128 sums in per-thread shared memory (libtim_cold: 126 regs,
# 4 blocks/SM; libtim_cold5: 96 regs, 5 blocks/SM, some spills) vs the kept build (libtim).
mkdir -p gpurun_out
for lib in libtim_cold libtim_cold5; do
  TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so timeout -s KILL 900 python -m pytest tests/test_gpu_ppo.py -m gpu -q -x 2>&1 | tail -1
done
for r in 1 2 3; do for lib in libtim libtim_cold libtim_cold5; do
  echo -n "ppo $r $lib "; TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so timeout -s KILL 300 python scripts/ppo_only.py $((1<<27)) | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print(round(d['achieved'],1),'GB/s', round(d['ms'],4),'ms')"
done; done
