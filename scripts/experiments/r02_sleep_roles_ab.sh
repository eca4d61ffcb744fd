#!/bin/bash
# Round 2 (late): mbarrier waits that sleep (suspend-time hint) per warp role -- bit 1 TMA producer,
# 2 epilogue, 4 MMA issuer -- for the sampling twin (C1, scripts/sample_only.py) and the log-prob
# step (C1, scripts/c2_steps.py CFG=c1): the spinning producer / MMA warps share SMSPs 0 / 1 with
# two of the four epilogue warps.  Interleaved x2.
for r in 1 2; do
  for sl in 0 1 4 5; do
    echo -n "$r sample sleep=$sl "; TUN=3,2,$sl,4 REPS=10 python scripts/sample_only.py
  done
  for sl in 0 5; do
    echo -n "$r logprob c1 sleep=$sl "; CFG=c1 TUN=3,2,$sl,4 python scripts/c2_steps.py 30 | tail -1
  done
done
