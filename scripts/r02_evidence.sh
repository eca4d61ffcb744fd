#!/bin/bash
# Round-2 evidence in one call: GPU tests, smoke, default bench line (C2 headline + C1/C3 extra
# configs), the launch list of a short bench run, ncu --set full of the C2 log-prob kernel, of the
# correction pass 1 and of the PPO pass at 2^27 tokens.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
timeout -s KILL 1800 python -m pytest tests -m gpu -q > gpurun_out/tests_gpu.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/tests_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-extra-configs --no-backward-bench \
   --no-sample-bench > gpurun_out/launches_bench.json 2>&1; echo ncu1_rc=$?
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:logprob_fwd -s 2 -c 1 \
   -o gpurun_out/prof_logprob_c2 -f python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
   --no-extra-configs --no-backward-bench --no-sample-bench --correction-tokens 0 > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
REPS=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:correct_local -s 3 -c 1 \
   -o gpurun_out/prof_correct -f python scripts/correct_only.py > gpurun_out/ncu_full_corr.log 2>&1; echo ncu3_rc=$?
REPS=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:ppo_local -s 3 -c 1 \
   -o gpurun_out/prof_ppo -f python scripts/ppo_only.py > gpurun_out/ncu_full_ppo.log 2>&1; echo ncu4_rc=$?
cat gpurun_out/bench.json
