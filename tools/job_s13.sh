#!/bin/bash
R=$PWD
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/t13.txt
bash tools/ab_ingest.sh "TWG_LIB_PATH=$R/build/ab/base.so" "TWG_LIB_PATH=$R/build/ab/stats2.so" "TWG_LIB_PATH=$R/build/ab/base.so" "TWG_LIB_PATH=$R/build/ab/stats2.so"
timeout 300 ncu --metrics launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_bucket_place -s 9 -c 1 --csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-audit 2>/dev/null | grep k_bucket_place | awk -F'","' '{print $(NF-2), $NF}' >> gpurun_out/ab_ingest.txt
cat gpurun_out/t13.txt >> gpurun_out/ab_ingest.txt
cat gpurun_out/ab_ingest.txt
