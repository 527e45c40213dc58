# e2e variance probe: three benches back to back, per-step e2e loop times
for i in 1 2 3; do
  TWG_BENCH_VERBOSE=1 python bench.py --no-cpu-baseline > gpurun_out/e2e$i.json 2>gpurun_out/e2e$i.err
  python -c "import json; d=json.load(open('gpurun_out/e2e$i.json')); print('run $i', round(d['value']/1e9,3), 'e2e', round(d['e2e']['value']/1e9,3))"
  grep "e2e step" gpurun_out/e2e$i.err | tr '\n' ' ' | sed 's/e2e step//g'; echo
done
