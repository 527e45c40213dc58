#!/bin/bash
# walk kernel cost by walk length (start only, +1 hop, ...): time and DRAM bytes per launch
mkdir -p gpurun_out
out=gpurun_out/walklen.txt; : > $out
for L in 2 3 4 5 80; do
  echo "== L $L" >> $out
  timeout 300 python tools/diag_walk.py 1.0 3 fullwalk $L 2>&1 | grep "rep 2" >> $out
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_fullwalk -s 1 -c 1 --csv python tools/diag_walk.py 1.0 2 fullwalk $L 2>/dev/null | grep k_fullwalk | awk -F'","' '{print $(NF-2), $NF}' >> $out
done
cat $out
