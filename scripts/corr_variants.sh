#!/bin/bash
# build correction-kernel variants (tokens per lane x min blocks per SM) and time each at 2^27 tokens
set -e
cd "$(dirname "$0")/.."
for v in ${CORR_VARIANTS:-4x3 4x2 8x2}; do
  tpl=${v%x*}; minb=${v#*x}
  out=/tmp/libtim_${tpl}_${minb}.so
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared --expt-relaxed-constexpr \
    -DTIM_CORR_TPL=$tpl -DTIM_CORR_MINB=$minb -I include -o $out paper_2605_14220_b200/csrc/{api,logprob,correct,ppo,rmsnorm}.cu -ldl
  echo "== tpl=$tpl minb=$minb"; TIM_LIBRARY=$out timeout 300 python scripts/correct_only.py $((1<<27)) | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print(round(d['achieved'],1),'GB/s', round(d['ms'],3),'ms')"
done
