#!/bin/bash
# A/B walk kernels across library builds: time (CUDA events) and ncu DRAM bytes per C5 launch
# usage: tools/ab_walklib.sh name1.so name2.so ...   (files under build/ab/)
mkdir -p gpurun_out
out=gpurun_out/ab_walklib.txt; : > $out
for rep in 1 2; do
for so in "$@"; do
  echo "== $so" >> $out
  TWG_LIB_PATH=$PWD/build/ab/$so timeout 300 python tools/diag_walk.py 1.0 4 2>&1 | grep -E "rep 3|rror" >> $out
  if [ $rep = 1 ]; then
  TWG_LIB_PATH=$PWD/build/ab/$so timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_fullwalk -s 1 -c 1 --csv python tools/diag_walk.py 1.0 2 2>/dev/null | grep k_fullwalk | awk -F'","' '{print $(NF-2), $NF}' >> $out
  fi
done
done
cat $out
