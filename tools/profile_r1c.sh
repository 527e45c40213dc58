#!/bin/bash
# Round-1 closing profile set: launch list of the C5 bench + full captures of
# the walk kernel and the steady-state ingest kernels.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r1c.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fullwalk -s 1 -c 1 \
  -o gpurun_out/r1c_fullwalk -f python tools/diag_walk.py 1.0 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_bucket_place|k_batch_stats|k_plan|k_radix_scatter|k_bucket_count|k_scan_scatter|k_reloc_copy" \
  -s 60 -c 10 -o gpurun_out/r1c_ingest -f python tools/diag_ingest.py 1.0 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/*.csv
