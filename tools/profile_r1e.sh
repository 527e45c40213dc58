#!/bin/bash
# Profile set after the walk-search / onesweep changes: launch list of the C5
# bench, full captures of the walk kernel, the radix passes and the
# placement/plan kernels (steady-state batches of tools/diag_ingest.py).
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r1e.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-audit > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fullwalk -s 1 -c 1 \
  -o gpurun_out/r1e_fullwalk -f python tools/diag_walk.py 1.0 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_bucket_place|k_batch_stats|k_plan|k_radix_onesweep|k_radix_global_hist|k_bucket_count|k_scan_scatter|k_reloc_copy" \
  -s 60 -c 10 -o gpurun_out/r1e_ingest -f python tools/diag_ingest.py 1.0 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/*.csv
