#!/bin/bash
# Full ncu captures of the top ingest kernels at C5 scale (one launch each, steady state).
tag=${1:-r1}
for k in "k_merge_tiles" "k_scan_scatter" ; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 20 -c 3 \
    -o gpurun_out/prof_${tag}_${k} -f python tools/diag_ingest.py 1.0 > /dev/null 2>&1
done
ls -la gpurun_out
