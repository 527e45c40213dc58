#!/bin/bash
R=$PWD
for so in head wrec; do
TWG_LIB_PATH=$R/build/ab/$so.so timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launch_$so.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-audit > /dev/null 2>&1
done
ls -la gpurun_out/launch_*
