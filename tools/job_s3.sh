#!/bin/bash
bash tools/ab_ingest.sh "TWG_STATS_GROUPS=1" "TWG_STATS_GROUPS=0" "TWG_COMPACT_PAYLOAD=0" 
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_bucket_place|k_batch_stats|k_radix_onesweep|k_bucket_count" \
  -s 40 -c 5 -o gpurun_out/s3_ingest -f python tools/diag_ingest.py 1.0 > gpurun_out/ncu_ingest3.log 2>&1
ls gpurun_out
