#!/bin/bash
# Round 2: with die-aware groups, C2 W-window slack {1, 2, 4 (default)} x group {2 (auto), 4}, full C2 batch, interleaved.
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for rep in 1 2; do
for t in default 3,2,0,2 3,2,0,1 3,2,0,4,4 3,2,0,2,4; do
  echo -n "$rep "; timeout -s KILL 600 python scripts/c2_diag.py 2097152 $t 3 | tail -1
done
done
