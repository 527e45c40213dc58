"""Per-CUDA-line summary of an ncu source page (--page source --csv --print-source cuda,sass):
warp-stall samples and L2 theoretical global sectors per source line, top N by a column.
usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > x.csv; python tools/ncu_src_lines.py x.csv [N] [col]"""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
key = sys.argv[3] if len(sys.argv) > 3 else "L2 Theoretical Sectors Global"
rows, hdr, fname = [], None, ""
for r in csv.reader(open(path)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name") or not r[0].isdigit():
        continue
    d = dict(zip(hdr[2:], r[2:]))
    def num(c):
        try:
            return float(d.get(c, "0").replace(",", ""))
        except ValueError:
            return 0.0
    rows.append((num(key), num("# Samples"), num("L2 Theoretical Sectors Global"), num("L1 Tag Requests Global"),
                 num("Instructions Executed"), f"{fname}:{r[0]}", r[1].strip()[:90]))
tot = [sum(x[i] for x in rows) for i in range(5)]
print(f"totals: samples {tot[1]:.0f}  L2 sectors {tot[2]:.4g}  L1 tag req {tot[3]:.4g}  warp inst {tot[4]:.4g}")
for x in sorted(rows, key=lambda x: -x[0])[:top]:
    print(f"{x[1]:7.0f} {100*x[1]/max(tot[1],1):5.1f}%  inst {x[4]:10.4g}  L2sec {x[2]:11.4g}  L1req {x[3]:10.4g}  {x[5]:18s} {x[6]}")
