#!/bin/bash
# Round 2 (late): correction pass 1 store / ring-depth variants in the hot loop (scripts/corr_time.py:
# whole tim_correct and pass 1 alone): libtim (st.global.cs stores, 4 stages), libtim_plain (plain
# stores), libtim_st5 (5-stage per-lane ring).
mkdir -p gpurun_out
TIM_LIBRARY=$PWD/paper_2605_14220_b200/libtim_plain.so timeout -s KILL 900 python -m pytest tests/test_gpu_correct.py -m gpu -q -x 2>&1 | tail -1
for r in 1 2 3; do for lib in libtim libtim_plain libtim_st5; do echo -n "$r $lib "; TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so python scripts/corr_time.py; done; done
