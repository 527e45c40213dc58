#!/bin/bash
# Run on the GPU box: launch list + one full ncu capture of the top kernels.
# usage: tools/profile_box.sh <tag> <scale>
tag=${1:-r1}; scale=${2:-0.1}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${tag}.csv python bench.py --scale $scale --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for k in k_fullwalk k_radix_scatter k_entries k_mark_present; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/prof_${tag}_${k} -f python tools/diag_walk.py $scale 1 > /dev/null 2>&1
done
ls -la gpurun_out
