#!/bin/bash
R=$PWD
bash tools/ab_ingest.sh "TWG_LIB_PATH=$R/build/ab/wrec.so" "TWG_LIB_PATH=$R/build/ab/wrec2.so" "TWG_LIB_PATH=$R/build/ab/head.so" "TWG_LIB_PATH=$R/build/ab/wrec2.so"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 >> gpurun_out/ab_ingest.txt
cat gpurun_out/ab_ingest.txt
