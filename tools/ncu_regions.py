"""Aggregate an ncu source page (--print-source cuda,sass --csv) into line-range regions.
  python tools/ncu_regions.py src.csv file.cu name:lo-hi name:lo-hi ..."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
target = sys.argv[2]
regions = []
for spec in sys.argv[3:]:
    name, rng = spec.split(":")
    lo, hi = map(int, rng.split("-"))
    regions.append((name, lo, hi))
hdr = None
fname = "?"
cur = None
R = defaultdict(lambda: [0.0, 0.0])
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        continue
    try:
        s = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        ie = float(r[hdr.index("Instructions Executed")] or 0)
    except ValueError:
        continue
    name = "other:" + cur[0]
    if cur[0] == target:
        name = "other"
        for n, lo, hi in regions:
            if lo <= cur[1] <= hi:
                name = n
                break
    R[name][0] += s
    R[name][1] += ie
ts = sum(v[0] for v in R.values()) or 1
ti = sum(v[1] for v in R.values()) or 1
print(f"total instructions {ti:.4g}")
for k, v in sorted(R.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:36s} instr {100 * v[1] / ti:5.1f}%   stall samples {100 * v[0] / ts:5.1f}%")
