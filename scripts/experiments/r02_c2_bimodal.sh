#!/bin/bash
# Round 2 (late): the C2 step-time bimodality (fast ~1.78 s / slow ~1.9-1.98 s launches) under L2
# knobs: default (H evict_last, W evict_first, slack 4), finished H tiles demoted to evict_normal,
# H evict_normal.  scripts/c2_steps.py: per-step log-prob kernel time, 12 steps per process.
for r in 1 2; do
  echo "== default"; python scripts/c2_steps.py 12 | tail -1
  echo "== demote"; DEMOTE=1 python scripts/c2_steps.py 12 | tail -1
  echo "== h_normal"; TUN=1,2,0,4 python scripts/c2_steps.py 12 | tail -1
done
