"""Per-CUDA-source-line executed instruction counts from an ncu
`--page source --csv --print-source cuda,sass` export (profiling aid).

  python scripts/src_lines.py export.csv n_points [top]
"""
import csv
import sys
from collections import defaultdict

n = float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
rows = list(csv.reader(open(sys.argv[1])))
path = None
per = defaultdict(lambda: [0.0, 0.0, defaultdict(float), ""])
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ix = hdr.index("Instructions Executed")
        isamp = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= ix:
        continue
    try:
        c = float(r[ix] or 0)
        s = float(r[isamp] or 0)
    except ValueError:
        continue
    if c == 0 and s == 0:
        continue
    key = (path, r[0])
    e = per[key]
    e[0] += c
    e[1] += s
    e[3] = r[1].strip()[:70]
tot = sum(v[0] for v in per.values())
ts = sum(v[1] for v in per.values())
print(f"total {tot / n:.1f} warp-instr/pt")
for (f, ln), v in sorted(per.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{f}:{ln:>5s} {v[0] / n:7.2f}/pt samp {100 * v[1] / ts:5.1f}%  {v[3]}")
