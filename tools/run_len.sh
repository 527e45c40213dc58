#!/bin/bash
# A/B: walk time by walk length (tools/diag_walk_len.py) per library build: tools/run_len.sh a.so b.so
for l in "$@"; do echo $l; TWG_LIB_PATH=$PWD/$l timeout 300 python tools/diag_walk_len.py 2>&1 | grep "L="; done
