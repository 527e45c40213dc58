#!/bin/bash
R=$PWD
bash tools/ab_walkenv.sh "TWG_LIB_PATH=$R/build/ab/base.so" "TWG_LIB_PATH=$R/build/ab/pair24.so" "TWG_LIB_PATH=$R/build/ab/pair20.so" "TWG_LIB_PATH=$R/build/ab/pair32.so"
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or walk or golden or facade or append or acceptance" 2>&1 | tail -2 >> gpurun_out/ab_walkenv.txt
cat gpurun_out/ab_walkenv.txt
