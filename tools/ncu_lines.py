"""Aggregate an ncu source page (--print-source cuda,sass --csv) per CUDA source line:
share of stall samples and of executed instructions, top stall reasons."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = defaultdict(lambda: [0.0, 0.0, defaultdict(float)])
fname = "?"
hdr = None
cur = None
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
    if r[0]:  # a CUDA source line row
        cur = (fname, r[0], r[1].strip()[:80])
        continue
    if cur is None:
        continue
    try:
        s = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        ie = float(r[hdr.index("Instructions Executed")] or 0)
    except ValueError:
        continue
    a = agg[cur]
    a[0] += s
    a[1] += ie
    for k, name in enumerate(hdr):
        if name.startswith("stall_") and "Not Issued" not in name:
            try:
                a[2][name] += float(r[k] or 0)
            except ValueError:
                pass
ts = sum(a[0] for a in agg.values()) or 1
ti = sum(a[1] for a in agg.values()) or 1
print(f"total stall samples {ts:.0f}, instructions {ti:.3g}")
for key, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    st = sorted(a[2].items(), key=lambda kv: -kv[1])[:3]
    sts = " ".join(f"{k[6:]}={v / max(a[0], 1):.0%}" for k, v in st)
    print(f"{100 * a[0] / ts:5.1f}% smp {100 * a[1] / ti:5.1f}% ins {key[0]}:{key[1]}: {key[2]}  [{sts}]")
