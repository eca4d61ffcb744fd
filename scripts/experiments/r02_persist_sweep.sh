#!/bin/bash
# Round 2 (late): persisting-L2 set-aside size sweep, C2 and C1 step times (scripts/c2_steps.py).
python scripts/die_map_print.py
for r in 1 2; do
  for mb in 0 24 40 48 64; do
    echo "== c2 persist $mb"; PERSIST=$mb python scripts/c2_steps.py 8 | grep -E "persisting|median"
  done
  for mb in 0 48 79; do
    echo "== c1 persist $mb"; CFG=c1 PERSIST=$mb python scripts/c2_steps.py 30 | grep -E "persisting|median"
  done
done
