#!/bin/bash
# Round 2 (final build): ncu --set full of the correction pass 1 (2^27 tokens) and of the sampling
# twin (C1), plus the sampling twin's hot-loop time.
mkdir -p gpurun_out
REPS=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:correct_local -s 3 -c 1 \
   -o gpurun_out/prof_correct -f python scripts/correct_only.py > gpurun_out/ncu_full_corr.log 2>&1; echo ncu_corr_rc=$?
REPS=1 timeout -s KILL 900 ncu --set full --clock-control none -k regex:logprob_fwd -s 2 -c 1 \
   -o gpurun_out/prof_sample -f python scripts/sample_only.py > gpurun_out/ncu_full_sample.log 2>&1; echo ncu_sample_rc=$?
REPS=10 python scripts/sample_only.py
