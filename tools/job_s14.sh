#!/bin/bash
R=$PWD
bash tools/ab_ingest.sh "TWG_LIB_PATH=$R/build/ab/base.so" "TWG_LIB_PATH=$R/build/ab/items6.so" "TWG_LIB_PATH=$R/build/ab/items12.so" "TWG_LIB_PATH=$R/build/ab/base.so" "TWG_LIB_PATH=$R/build/ab/items6.so" "TWG_LIB_PATH=$R/build/ab/items12.so"
