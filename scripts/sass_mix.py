"""Dynamic SASS opcode mix from an ncu source-page export (test/profiling aid).

  ncu -i rep.ncu-rep --page source --csv --print-source sass > src.csv
  python scripts/sass_mix.py src.csv [n_points]
"""
import csv
import re
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = hdr.index("Instructions Executed")
isamp = hdr.index("Warp Stall Sampling (All Samples)")
n = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
mix, samp = Counter(), Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= ix:
        continue
    src = r[1].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", src)
    if not m:
        continue
    op = m.group(2)
    try:
        c = float(r[ix])
        s = float(r[isamp] or 0)
    except ValueError:
        continue
    mix[op] += c
    samp[op] += s
    tot += c
ts = sum(samp.values())
print(f"total warp instr {tot:.4g}  per point {tot / n:.1f}")
for op, c in mix.most_common(40):
    print(f"{op:10s} {c / n:9.2f} /pt  {100 * c / tot:5.1f}%   stall-samples {100 * samp[op] / max(ts, 1):5.1f}%")
