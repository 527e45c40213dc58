#!/bin/bash
# Round-2 profile set: launch list of the C5 bench (one steady-state step per
# kernel), full captures of the walk kernel and of the steady-state ingest
# kernels.  usage: tools/profile_r2.sh <tag>
tag=${1:-r2}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${tag}.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-audit > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fullwalk -s 1 -c 1 \
  -o gpurun_out/${tag}_fullwalk -f python tools/diag_walk.py 1.0 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_bucket_place|k_batch_stats|k_plan|k_radix_onesweep|k_radix_global_hist|k_bucket_count|k_scan_scatter|k_reloc_copy|k_lb_time|k_count_dead" \
  -s 60 -c 12 -o gpurun_out/${tag}_ingest -f python tools/diag_ingest.py 1.0 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/*.csv
