#!/bin/bash
R=$PWD
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/t20.txt
bash tools/ab_ingest.sh "TWG_LIB_PATH=$R/build/ab/base.so" "TWG_LIB_PATH=$R/build/ab/grec.so" "TWG_LIB_PATH=$R/build/ab/base.so" "TWG_LIB_PATH=$R/build/ab/grec.so"
for so in base grec; do
TWG_LIB_PATH=$R/build/ab/$so.so timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fullwalk -s 1 -c 1 --csv python tools/diag_walk.py 1.0 2 2>/dev/null | grep k_fullwalk | awk -F'","' '{print $(NF-2), $NF}' >> gpurun_out/ab_ingest.txt
done
cat gpurun_out/t20.txt >> gpurun_out/ab_ingest.txt
