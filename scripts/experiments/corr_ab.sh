#!/bin/bash
# A/B the correction kernel builds: parity tests on the default build, then 2^27-token timings,
# the launch list of one standalone tim_correct and one ncu --set full capture of pass 1.
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_correct.py tests/test_gpu_sweep.py -m gpu -q -x > gpurun_out/corr_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/corr_tests.log
for lib in paper_2605_14220_b200/libtim*.so; do
  echo "== $lib"
  for i in 1 2; do TIM_LIBRARY=$PWD/$lib timeout -s KILL 300 python scripts/correct_only.py $((1<<27)) | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print(round(d['achieved'],1),'GB/s', round(d['ms'],4),'ms')"; done
done
REPS=1 timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/corr_launches.csv python scripts/correct_only.py > /dev/null 2>&1; echo ncu1_rc=$?
REPS=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:correct_local -s 3 -c 1 \
   -o gpurun_out/prof_correct -f python scripts/correct_only.py > gpurun_out/ncu_corr.log 2>&1; echo ncu_rc=$?
