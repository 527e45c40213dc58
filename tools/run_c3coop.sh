#!/bin/bash
# A/B: C3 walks (FullWalk + Coop, tools/bench_configs.py) per library build: tools/run_c3coop.sh a.so b.so
for l in "$@"; do echo $l; TWG_LIB_PATH=$PWD/$l timeout 300 python tools/bench_configs.py C3 2>/dev/null | grep walks; done
