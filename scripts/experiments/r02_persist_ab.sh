#!/bin/bash
# Round 2 (late): default persisting-L2 set-aside (queried) vs 48 MB (-> 55 MB granted), interleaved
# x4 on a fresh box, C2 step times (scripts/c2_steps.py, 10 steps per process).
python scripts/die_map_print.py
for r in 1 2 3 4; do
  echo "== default"; QUERY=1 python scripts/c2_steps.py 10 | grep -E "median"
  echo "== 48 MB"; PERSIST=48 python scripts/c2_steps.py 10 | grep -E "median"
done
