#!/bin/bash
# Round evidence in one call: GPU tests, smoke, bench line, launch list, ncu --set full of the
# logprob, correction and PPO kernels.
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -m gpu -q > gpurun_out/tests_gpu.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/tests_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout -s KILL 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --correction-tokens 0 > gpurun_out/launches_bench.json 2>&1; echo ncu1_rc=$?
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:logprob_fwd -s 2 -c 1 \
   -o gpurun_out/prof_logprob -f python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --correction-tokens 0 > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
REPS=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:correct_local -s 3 -c 1 \
   -o gpurun_out/prof_correct -f python scripts/correct_only.py > gpurun_out/ncu_full_corr.log 2>&1; echo ncu3_rc=$?
REPS=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:ppo_local -s 3 -c 1 \
   -o gpurun_out/prof_ppo -f python scripts/ppo_only.py > gpurun_out/ncu_full_ppo.log 2>&1; echo ncu4_rc=$?
cat gpurun_out/bench.json
