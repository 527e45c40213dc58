#!/bin/bash
# Closing profile set: launch list of the C5 bench, then full captures of the
# LAST step's walk kernel and steady-state ingest kernels (skip counts derived
# from the launch list), and the driver-contract bench line.
# usage: tools/profile_r2g.sh <tag>
tag=${1:-r2g}
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-audit"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_launches.csv $CMD > /dev/null 2>&1
RE="k_bucket_place|k_batch_stats|k_plan|k_radix_onesweep|k_radix_global_hist|k_bucket_count|k_bucket_bounds|k_fullwalk"
read SKIP CNT < <(python - "$RE" gpurun_out/${tag}_launches.csv <<'PY'
import csv, re, sys
pat = re.compile(sys.argv[1]); seen = set(); names = []
for r in csv.DictReader(l for l in open(sys.argv[2]) if l.startswith('"')):
    if r["ID"] in seen: continue
    seen.add(r["ID"]); names.append(r["Kernel Name"])
last = max(i for i, n in enumerate(names) if "k_init_scalars" in n)
m = [i for i, n in enumerate(names) if pat.search(n.split("(")[0])]
print(sum(1 for i in m if i < last), sum(1 for i in m if i >= last))
PY
)
echo "skip $SKIP count $CNT" > gpurun_out/${tag}_capture.txt
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$RE" -s $SKIP -c $CNT \
  -o gpurun_out/${tag}_step -f $CMD > /dev/null 2>&1
python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
ls -la gpurun_out/${tag}*
