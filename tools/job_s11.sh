#!/bin/bash
R=$PWD
bash tools/ab_ingest.sh "TWG_LIB_PATH=$R/build/ab/statstma.so" "TWG_LIB_PATH=$R/build/ab/histfuse.so" "TWG_LIB_PATH=$R/build/ab/statstma.so" "TWG_LIB_PATH=$R/build/ab/histfuse.so"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 >> gpurun_out/ab_ingest.txt
cat gpurun_out/ab_ingest.txt
