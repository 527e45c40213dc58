#!/bin/bash
R=$PWD
bash tools/ab_walkenv.sh "TWG_LIB_PATH=$R/build/ab/base.so" "TWG_LIB_PATH=$R/build/ab/zf.so"
for so in base zf; do
TWG_LIB_PATH=$R/build/ab/$so.so timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fullwalk -s 1 -c 1 --csv python tools/diag_walk.py 1.0 2 2>/dev/null | grep k_fullwalk | awk -F'","' '{print $(NF-2), $NF}' >> gpurun_out/ab_walkenv.txt
done
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or walk or golden or facade or append or ref_suites or acceptance" 2>&1 | tail -2 >> gpurun_out/ab_walkenv.txt
cat gpurun_out/ab_walkenv.txt
