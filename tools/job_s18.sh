#!/bin/bash
R=$PWD
bash tools/ab_walkenv.sh "TWG_LIB_PATH=$R/build/ab/base.so" "TWG_LIB_PATH=$R/build/ab/wn48.so" "TWG_LIB_PATH=$R/build/ab/wn56.so"
