#!/bin/bash
mkdir -p gpurun_out
REPS=1 timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:correct_local -s 1 -c 1 -o gpurun_out/prof_correct -f python scripts/correct_only.py > gpurun_out/ncu_corr_full.log 2>&1; echo rc=$?
