#!/bin/bash
# correctness of the append-route tests, then bench A/B over env knobs (device-resident step only)
mkdir -p gpurun_out
out=gpurun_out/ab_ingest.txt; : > $out
timeout 900 python -m pytest tests -m gpu -x -q -k "append or parity or golden or group" 2>&1 | tail -3 >> $out
for envs in "$@"; do
  echo "== $envs" >> $out
  env $envs timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-audit 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
  l=l.strip()
  if not l.startswith('{'): continue
  d=json.loads(l); p=d['phases']
  print('ms/step %.3f ingest %.3f walk %.3f value %.4g' % (d['ms_per_step'], p['ingest_ms_per_step'], p['walk_ms_per_step'], d['value']))
" >> $out
done
cat $out
