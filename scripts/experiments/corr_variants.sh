#!/bin/bash
# build correction-kernel variants (min resident blocks per SM) and time each at 2^27 tokens
set -e
cd "$(dirname "$0")/.."
for minb in ${CORR_MINB:-3 2 4}; do
  out=/tmp/libtim_minb_${minb}.so
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared --expt-relaxed-constexpr \
    -DTIM_CORR_MINB=$minb -I include -o $out paper_2605_14220_b200/csrc/{api,logprob,correct,ppo,rmsnorm}.cu -ldl
  echo "== minb=$minb"; TIM_LIBRARY=$out timeout 300 python scripts/correct_only.py $((1<<27)) | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print(round(d['achieved'],1),'GB/s', round(d['ms'],3),'ms')"
done
