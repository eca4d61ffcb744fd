#!/bin/bash
# PPO kernel block-shape variants at 2^27 tokens
for lib in paper_2605_14220_b200/libtim*.so; do
  for i in 1 2; do TIM_LIBRARY=$PWD/$lib timeout -s KILL 300 python scripts/ppo_only.py $((1<<27)) | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read().strip().splitlines()[-1]); print('$lib', round(d['achieved'],1),'GB/s', round(d['ms'],4),'ms')"; done
done
