"""Replicated-tree partition (SURVEY 8(e) variant (i), bt_set_partition) on
one B200: the search time of every part p of P for P in (1, 2, 4, 8), one
after the other on the same GPU (each part is what rank p would run; no rank
waits on another).  A P-GPU step would take broadcast + build + max_p search.

  python tools/part_case.py [--config 5] [--reps 3] [--out profiles/...json]
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
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--out", default=None)
args = ap.parse_args()

pos_np, h_np = datagen.make_config(args.config, n=args.n)
n = pos_np.shape[0]
dev = torch.device("cuda:0")
pos = torch.from_numpy(pos_np).to(dev)
h = torch.from_numpy(h_np).to(dev)
counts = torch.empty(n, dtype=torch.int32, device=dev)
offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
nbr = torch.empty(n * datagen.NGMAX, dtype=torch.int32, device=dev)


def timed(fn):
    ts = []
    for r in range(args.reps + 1):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if r:
            ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


build_ms = timed(lambda: P.Tree(pos, datagen.BUCKET_SIZE, datagen.MAX_EMPTY).free())
t = P.Tree(pos, datagen.BUCKET_SIZE, datagen.MAX_EMPTY)
rows = []
for nparts in (1, 2, 4, 8):
    parts = []
    for p in range(nparts):
        t.set_partition(p, nparts)
        ms = timed(lambda: t.find_neighbors(h, datagen.NGMAX, counts=counts, offsets=offsets, nbr_idx=nbr))
        parts.append({"part": p, "search_ms": ms, "pairs": int(offsets[-1].item())})
    mx = max(q["search_ms"] for q in parts)
    mean = sum(q["search_ms"] for q in parts) / nparts
    rows.append({"nparts": nparts, "max_search_ms": mx, "mean_search_ms": mean, "imbalance": mx / mean,
                 "parts": parts})
t.free()
out = {"config": args.config, "n": n, "build_ms": build_ms, "device": torch.cuda.get_device_name(0),
       "pos_h_bytes": n * 32, "rows": rows}
text = json.dumps(out, indent=1)
print(text)
if args.out:
    open(args.out, "w").write(text + "\n")
