#!/bin/bash
# Round-2 check: GPU tests, V=1 partials, epilogue A/B (round-1 FFMA vs subtract-then-scale), bench line.
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x > gpurun_out/tests_gpu.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/tests_gpu.log
timeout 120 python scripts/dbg/v1_partials.py > gpurun_out/v1.txt 2>&1
bash scripts/experiments/lib_ab.sh > gpurun_out/epi_ab.txt 2>&1
timeout -s KILL 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
