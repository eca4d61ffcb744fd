#!/bin/bash
# Round 2 (late): correction pass 1 variants (libtim.so) vs the previous build (libtim_old.so);
# variant 3: the running max |delta| of the fast body as compare-and-select (no fmax NaN handling);
# correction parity first, then interleaved end-to-end timing at 2^27 tokens.
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests/test_gpu_correct.py tests/test_gpu_correct_paths.py tests/test_gpu_sweep.py tests/test_gpu_robustness.py -m gpu -q -x > gpurun_out/corr_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/corr_tests.log
for rep in 1 2 3; do
for lib in libtim_old libtim; do
  echo -n "$rep $lib "; TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so timeout -s KILL 300 python scripts/correct_only.py $((1<<27)) | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print(round(d['achieved'],1),'GB/s', round(d['ms'],4),'ms')"
done
done
REPS=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:correct_local -s 3 -c 1 \
   -o gpurun_out/prof_correct -f python scripts/correct_only.py > gpurun_out/ncu_full_corr.log 2>&1; echo ncu_rc=$?
