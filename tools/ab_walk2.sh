#!/bin/bash
# A/B of the FullWalk launch knobs on the C5 window (scale 1.0): block size,
# last_t terminal filter, L2 evict_last hint on the last_t loads.
mkdir -p gpurun_out
out=gpurun_out/ab_walk2.txt; : > $out
for cfg in "256 0 0" "256 1 0" "32 0 0" "32 1 0" "64 1 0" "128 1 0" "32 1 1" "64 1 1"; do
  set -- $cfg
  echo "== block $1 lastt $2 l2keep $3" >> $out
  TWG_WALK_BLOCK=$1 TWG_WALK_LASTT=$2 TWG_WALK_L2KEEP=$3 timeout 300 python tools/diag_walk.py 1.0 5 2>&1 | grep -E "rep|error|Error" >> $out
done
cat $out
