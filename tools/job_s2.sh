mkdir -p gpurun_out
./build/diag_accum 3 > gpurun_out/accum.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fullwalk -s 1 -c 1 \
  -o gpurun_out/s2_fullwalk -f python tools/diag_walk.py 1.0 2 > gpurun_out/ncu_walk.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_bucket_place|k_batch_stats|k_plan|k_radix_onesweep|k_scan_scatter" \
  -s 40 -c 6 -o gpurun_out/s2_ingest -f python tools/diag_ingest.py 1.0 > gpurun_out/ncu_ingest.log 2>&1
ls -la gpurun_out
