#!/bin/bash
# Round-1 profile set: launch list of the C5 bench + full captures of the top kernels.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r1_final.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fullwalk -s 1 -c 1 \
  -o gpurun_out/r1_fullwalk -f python tools/diag_walk.py 1.0 2 > /dev/null 2>&1
for k in k_scan_scatter k_place_x k_radix_scatter k_place_y_sorted k_copy_survivors; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 12 -c 2 \
    -o gpurun_out/r1_$k -f python tools/diag_ingest.py 1.0 > /dev/null 2>&1
done
ls -la gpurun_out/*.ncu-rep gpurun_out/*.csv
