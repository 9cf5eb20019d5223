"""Summarise tools/gpu_ab.sh outputs: per variant and round, the per-rep phase times."""
import glob
import json
import sys

for f in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab_*_r*.json")):
    s = open(f).read()
    try:
        d = json.loads(s[s.index("{"):])
    except ValueError:
        print(f, "unparsable", s[-200:])
        continue
    keys = ["search.desc", "search.count", "search.fill", "search.total", "build.total"]
    print(f.split("/")[-1].ljust(28), " | ".join(k.split(".")[1] + " " + " ".join(f"{r.get(k, 0):7.3f}" for r in d["per_rep"]) for k in keys))
