#!/bin/bash
# Round 2 (late): C2 step times (scripts/c2_steps.py, 10 steps per process) under L2 policy / demote
# combinations: TUN = h_policy,w_policy,sleep,slack (1 normal, 2 evict_first, 3 evict_last).
python scripts/die_map_print.py
for r in 1 2; do
  echo "== default (3,2,0,4)"; python scripts/c2_steps.py 10 | tail -1
  echo "== demote"; DEMOTE=1 python scripts/c2_steps.py 10 | tail -1
  echo "== demote + W normal"; DEMOTE=1 TUN=3,1,0,4 python scripts/c2_steps.py 10 | tail -1
  echo "== W normal"; TUN=3,1,0,4 python scripts/c2_steps.py 10 | tail -1
  echo "== demote + W last"; DEMOTE=1 TUN=3,3,0,4 python scripts/c2_steps.py 10 | tail -1
done
