#!/bin/bash
R=$PWD
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/t17.txt
bash tools/ab_ingest.sh "TWG_LIB_PATH=$R/build/ab/base.so" "TWG_LIB_PATH=$R/build/ab/evict.so" "TWG_LIB_PATH=$R/build/ab/base.so" "TWG_LIB_PATH=$R/build/ab/evict.so"
cat gpurun_out/t17.txt >> gpurun_out/ab_ingest.txt
