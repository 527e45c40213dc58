#!/bin/bash
# A/B of walk-kernel env knobs on the C5 window: CUDA-event time per launch (rep 3 of 4)
mkdir -p gpurun_out
out=gpurun_out/ab_walkenv.txt; : > $out
for rep in 1 2; do
for envs in "$@"; do
  echo "== $envs" >> $out
  env $envs timeout 300 python tools/diag_walk.py 1.0 4 2>&1 | grep -E "rep 3|rror" >> $out
done
done
cat $out
