#!/bin/bash
# packed fp32 (FFMA2 / FADD2) epilogues: GPU tests, bitwise digests of both builds, interleaved timings
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for lib in libtim_old libtim; do echo -n "$lib "; TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so timeout -s KILL 300 python scripts/digest.py; done
bash scripts/experiments/lib_ab.sh
bash scripts/experiments/bwd_ab.sh
