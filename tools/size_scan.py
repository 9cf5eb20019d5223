"""Throughput against problem size on one B200: the cfg 5 recipe at
N = 2^22 .. 2^26 (h rescaled as N^(-1/3) by make_config), build + count + exact
fill (count-only call, exact CSR allocation, fill-only call), CUDA events.

  python tools/size_scan.py [--out profiles/...json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1910_02639_b200 as P  # noqa: E402
from paper_1910_02639_b200 import datagen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=None)
ap.add_argument("--max-log2", type=int, default=26)
ap.add_argument("--min-log2", type=int, default=22)
args = ap.parse_args()
dev = torch.device("cuda:0")
rows = []
for lg in range(args.min_log2, args.max_log2 + 1):
    n = 1 << lg
    pos_np, h_np = datagen.make_config(5, n=n)
    pos, h = torch.from_numpy(pos_np).to(dev), torch.from_numpy(h_np).to(dev)
    del pos_np, h_np
    ts = []
    for r in range(3):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        t = P.Tree(pos, 64, 0.5)
        c, o = t.count(h)
        nbr = t.fill(h, o)
        b.record()
        torch.cuda.synchronize()
        st = t.stats()
        t.free()
        del c, o, nbr
        if r:
            ts.append(a.elapsed_time(b))
    ms = min(ts)
    rows.append({"n": n, "ms": ms, "particles_per_s": n / (ms * 1e-3), "pairs": st["total_pairs"],
                 "pairs_per_s": st["total_pairs"] / (ms * 1e-3), "max_count": st["max_count"],
                 "torch_peak_gb": torch.cuda.max_memory_allocated() / 1e9})  # inputs + CSR (the library's own blocks not included)
    print(json.dumps(rows[-1]), flush=True)
    del pos, h
    torch.cuda.empty_cache()
    P.release_cache()
out = {"device": torch.cuda.get_device_name(0), "recipe": "cfg 5 (make_config(5, n))", "rows": rows}
if args.out:
    open(args.out, "w").write(json.dumps(out, indent=1) + "\n")
