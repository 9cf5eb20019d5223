"""Run build + find_neighbors on one config a few times and print phase times
(library CUDA events).  Used for ncu captures and quick timing on the box."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1910_02639_b200 as P  # noqa: E402
from paper_1910_02639_b200 import datagen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--exact", action="store_true")
ap.add_argument("--ngmax", type=int, default=512)
ap.add_argument("--count-only", action="store_true")
ap.add_argument("--symmetric", action="store_true", help="max(h_i, h_j) criterion (bt_find_neighbors_sym)")
ap.add_argument("--tree-order", action="store_true", help="bt_set_tree_order: h by tree position (bt_reorder)")
args = ap.parse_args()

pos_np, h_np = datagen.make_config(args.config, n=args.n)
n = pos_np.shape[0]
dev = torch.device("cuda:0")
pos = torch.from_numpy(pos_np).to(dev)
h = torch.from_numpy(h_np).to(dev)
counts = torch.empty(n, dtype=torch.int32, device=dev)
offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
nbr = torch.empty(n * args.ngmax, dtype=torch.int32, device=dev)
P.set_exact_only(args.exact)
per_rep = []
for r in range(args.reps):
    P.profile_reset()
    P.profile_enable(True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    t = P.Tree(pos, 64, 0.5)
    hq = h
    if args.tree_order:
        t.set_tree_order(True)
        hq = t.reorder(h)
    if args.count_only:
        t.count(hq, symmetric=args.symmetric)
    else:
        t.find_neighbors(hq, args.ngmax, counts=counts, offsets=offsets, nbr_idx=nbr, symmetric=args.symmetric)
    st = t.stats()
    t.free()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    per_rep.append({k: round(v[0], 3) for k, v in P.profile().items() if k.startswith("search.") or k == "build.total"})
prof = P.profile()
print(json.dumps({"n": n, "wall_ms_last": (t1 - t0) * 1e3, "stats": st, "per_rep": per_rep,
                  "phases_ms": {k: round(v[0], 4) for k, v in prof.items() if not k.startswith("kernel.")},
                  "launches": {k: v[1] for k, v in prof.items() if k.startswith("kernel.")}}, indent=1))
