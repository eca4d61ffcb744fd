#!/bin/bash
# Round 2 (late): C2 step times vs the progress-gate slack (scripts/c2_steps.py, 10 steps per process).
python scripts/die_map_print.py
for r in 1 2; do
  for t in 3,2,0,4 3,2,0,2 3,2,0,1 3,2,0,8; do echo "== TUN=$t"; TUN=$t python scripts/c2_steps.py 10 | tail -1; done
done
