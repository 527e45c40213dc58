#!/bin/bash
R=$PWD
bash tools/ab_ingest.sh "TWG_LIB_PATH=$R/build/ab/stat6.so" "TWG_LIB_PATH=$R/build/ab/stat4.so" "TWG_LIB_PATH=$R/build/ab/stat6.so" "TWG_LIB_PATH=$R/build/ab/stat4.so"
