#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > gpurun_out/t4.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/t4.log
bash scripts/ncu_variants.sh
