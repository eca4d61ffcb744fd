#!/bin/bash
for rep in 1 2 3; do
for lib in libtim_old libtim; do
  TIM_LIBRARY=$PWD/paper_2605_14220_b200/$lib.so timeout -s KILL 300 python scripts/sample_only.py | sed "s/^/$rep $lib /"
done
done
