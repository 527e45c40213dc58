#!/bin/bash
R=$PWD
bash tools/ab_ingest.sh "TWG_LIB_PATH=$R/build/ab/base.so" "TWG_LIB_PATH=$R/build/ab/pent4.so" "TWG_LIB_PATH=$R/build/ab/pent5_1792.so" "TWG_LIB_PATH=$R/build/ab/pent5_1536.so" "TWG_LIB_PATH=$R/build/ab/base.so" "TWG_LIB_PATH=$R/build/ab/pent4.so" "TWG_LIB_PATH=$R/build/ab/pent5_1792.so" "TWG_LIB_PATH=$R/build/ab/pent5_1536.so"
