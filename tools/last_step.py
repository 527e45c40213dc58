"""Per-kernel table of the LAST bench step from an ncu --csv launch list
(--metrics gpu__time_duration.sum[,dram__bytes_read.sum,dram__bytes_write.sum]):
the launches from the last k_init_scalars through the last k_fullwalk.
usage: python tools/last_step.py launches.csv [launches2.csv]"""
import csv
import sys


def load(path):
    rows = {}
    order = []
    for r in csv.DictReader(l for l in open(path) if l.startswith('"')):
        key = r["ID"]
        if key not in rows:
            rows[key] = {"name": r["Kernel Name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")}
            order.append(key)
        v = r["Metric Value"].replace(",", "")
        rows[key][r["Metric Name"]] = float(v) if v else 0.0
    seq = [rows[k] for k in order]
    last_walk = max(i for i, x in enumerate(seq) if "k_fullwalk" in x["name"])
    first = max(i for i, x in enumerate(seq[:last_walk]) if "k_init_scalars" in x["name"])
    return seq[first:last_walk + 1]


tabs = [load(p) for p in sys.argv[1:]]
for p, t in zip(sys.argv[1:], tabs):
    tot = sum(x.get("gpu__time_duration.sum", 0) for x in t) / 1e3
    print(f"== {p}: {len(t)} launches, {tot:.1f} us")
    for x in t:
        us = x.get("gpu__time_duration.sum", 0) / 1e3
        rd = x.get("dram__bytes_read.sum", 0) / 1e9
        wr = x.get("dram__bytes_write.sum", 0) / 1e9
        print(f"  {x['name'][:70]:70s} {us:9.1f} us  R {rd:6.3f} GB  W {wr:6.3f} GB")
