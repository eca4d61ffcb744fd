#!/bin/bash
# Round 2 (late): L2 hints of the HBM-bound passes.  Correction (scripts/corr_time.py): libtim (plain
# stores, evict_first cp.async reads), libtim_czp (+ plain stores in the zeroing pass), libtim_cnh
# (reads without the evict_first policy).  PPO (scripts/ppo_only.py): libtim (st.global.cs stores),
# libtim_pp (plain stores), libtim_pnh (reads without the evict_first policy).
mkdir -p gpurun_out
for r in 1 2 3; do for lib in libtim libtim_czp libtim_cnh; do echo -n "corr $r $lib "; TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so python scripts/corr_time.py; done; done
for r in 1 2 3; do for lib in libtim libtim_pp libtim_pnh; do
  echo -n "ppo $r $lib "; TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so timeout -s KILL 300 python scripts/ppo_only.py $((1<<27)) | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print(round(d['achieved'],1),'GB/s', round(d['ms'],4),'ms')"
done; done
