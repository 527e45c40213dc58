#!/bin/bash
# A/B the walk phase of the C5 bench across library builds: tools/ab_walk.sh a.so b.so ...
for rep in 1 2 3 4; do
  for lib in "$@"; do
    TWG_LIB_PATH=$PWD/$lib python bench.py --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); p=d['phases']
print('$lib', round(d['ms_per_step'],3), 'ingest', round(p['ingest_ms_per_step'],3), 'walk', round(p['walk_ms_per_step'],3))"
  done
done
