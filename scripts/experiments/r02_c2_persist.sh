#!/bin/bash
# Round 2 (late): C2 step times with the device's persisting-L2 set-aside raised (the evict_last H
# tiles) vs the default (0), scripts/c2_steps.py, 10 steps per process.
python scripts/die_map_print.py
for r in 1 2; do
  echo "== default"; python scripts/c2_steps.py 10 | tail -1
  echo "== persist 96 MB"; PERSIST=96 python scripts/c2_steps.py 10 | grep -E "persisting|median"
  echo "== persist 48 MB"; PERSIST=48 python scripts/c2_steps.py 10 | grep -E "persisting|median"
done
