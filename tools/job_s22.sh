#!/bin/bash
R=$PWD
bash tools/ab_ingest.sh "TWG_LIB_PATH=$R/build/ab/base.so" "TWG_LIB_PATH=$R/build/ab/evict2.so" "TWG_LIB_PATH=$R/build/ab/base.so" "TWG_LIB_PATH=$R/build/ab/evict2.so"
