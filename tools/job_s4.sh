#!/bin/bash
R=$PWD
bash tools/ab_ingest.sh "TWG_LIB_PATH=$R/build/ab/head.so" "TWG_LIB_PATH=$R/build/ab/bitmask.so" "TWG_LIB_PATH=$R/build/ab/head.so" "TWG_LIB_PATH=$R/build/ab/bitmask.so"
bash tools/job_walklen.sh
