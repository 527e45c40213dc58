#!/bin/bash
mkdir -p gpurun_out
bash tools/ab_ingest.sh "TWG_WALK_REC=1" "TWG_WALK_REC=0" "TWG_WALK_REC=1"
for r in 1 0; do
TWG_WALK_REC=$r timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_fullwalk -s 1 -c 1 --csv python tools/diag_walk.py 1.0 2 2>/dev/null | grep k_fullwalk | awk -F'","' '{print $(NF-2), $NF}' >> gpurun_out/ab_ingest.txt
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 >> gpurun_out/ab_ingest.txt
cat gpurun_out/ab_ingest.txt
