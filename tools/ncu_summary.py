#!/usr/bin/env python3
"""Summarise an ncu launch list (gpu__time_duration.sum CSV) and full
captures (.ncu-rep) into markdown for profiles/.

usage: tools/ncu_summary.py <launches.csv> [prof1.ncu-rep ...] > profiles/<name>.md
"""
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads per instruction (warp efficiency, /32)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "stall long_scoreboard"),
]


def to_us(v, unit):
    v = float(v.replace(",", ""))
    return {"ns": v / 1e3, "nsecond": v / 1e3, "us": v, "usecond": v, "ms": v * 1e3, "msecond": v * 1e3}.get(unit, v)


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("twg::<unnamed>::", "").replace("<unnamed>::", "").replace("twg::", "")
        us = to_us(r[vi], r[ui])
        agg[name][0] += 1
        agg[name][1] += us
        tot += us
    out = ["| kernel | launches | total µs | share |", "|---|---:|---:|---:|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
        out.append(f"| `{k}` | {n} | {t:,.1f} | {100 * t / tot:.1f}% |")
    out.append(f"| **total** | {sum(n for n, _ in agg.values())} | {tot:,.1f} | 100% |")
    return "\n".join(out)


def capture(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return f"(no data in {path})"
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        out.append(f"**{name.split('(')[0]}** (`{path.split('/')[-1]}`)\n")
        out.append("| metric | value |\n|---|---:|")
        for m, label in METRICS:
            if m in hdr:
                i = hdr.index(m)
                out.append(f"| {label} (`{m}`) | {vals[i]} {units[i]} |")
        out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    print("## Launch list (ncu gpu__time_duration.sum, cold-cache, serialised)\n")
    print(launches(sys.argv[1]))
    for p in sys.argv[2:]:
        print("\n## Full capture\n")
        print(capture(p))
