#!/bin/bash
# Round 2 (late): is it the set-aside size or the act of setting the persisting-L2 limit?  Default
# (limit only queried), explicit 0, 40 MB; C2 step times (scripts/c2_steps.py), 10 steps per process.
python scripts/die_map_print.py
for r in 1 2 3; do
  echo "== query only"; QUERY=1 python scripts/c2_steps.py 10 | grep -E "persisting|median"
  echo "== explicit 0"; PERSIST=0 python scripts/c2_steps.py 10 | grep -E "persisting|median"
  echo "== 40 MB"; PERSIST=40 python scripts/c2_steps.py 10 | grep -E "persisting|median"
done
