"""Bucket-size / beta sweeps and the b-tree vs octree comparison on one B200.

SURVEY 8(f) "next" rows 1-2: the paper's Sec. IV-B (b-tree vs octree build and
search), Sec. IV-C (bucket size s) and Sec. IV-D (beta,
P:463-476), measured on the synthetic BASELINE.json configurations instead of
the EC/SP snapshots.  Every setting must give the same neighbor counts (the
result does not depend on the tree): the sweep checks a checksum of the count
array against the first setting and records it.

  python tools/sweep.py --config 2 [--n N] [--reps 3] [--out profiles/...json]
"""
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
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--ngmax", type=int, default=512)
ap.add_argument("--plane", type=int, default=0,
                help="planar input of this many particles (z = 0, ~100 2-D neighbours) instead of a config")
ap.add_argument("--out", default=None)
args = ap.parse_args()

if args.plane:
    import numpy as np
    rng = np.random.default_rng(7)
    pos_np = np.zeros((args.plane, 3))
    pos_np[:, :2] = rng.random((args.plane, 2))
    h_np = 0.5 * np.sqrt(100.0 / (np.pi * args.plane)) * rng.uniform(0.8, 1.2, args.plane)
else:
    pos_np, h_np = datagen.make_config(args.config, n=args.n)
n = pos_np.shape[0]
dev = torch.device("cuda:0")
pos = torch.from_numpy(pos_np).to(dev)
h = torch.from_numpy(h_np).to(dev)
counts = torch.empty(n, dtype=torch.int32, device=dev)
offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
nbr = torch.empty(n * args.ngmax, dtype=torch.int32, device=dev)
weights = torch.arange(1, n + 1, dtype=torch.int64, device=dev)


def run(s, beta, policy):
    """Median over reps of (build ms, search ms) with CUDA events on the library
    stream (bt_profile phases), plus tree statistics and a count checksum."""
    builds, searches = [], []
    st = None
    for r in range(args.reps + 1):
        P.profile_reset()
        P.profile_enable(True)
        t = P.build(pos, s, beta, policy=policy)
        t.find_neighbors(h, args.ngmax, counts=counts, offsets=offsets, nbr_idx=nbr)
        st = t.stats()
        t.free()
        P.profile_enable(False)
        prof = P.profile()
        if r > 0:  # first run: warm-up
            builds.append(prof["build.total"][0])
            searches.append(prof["search.total"][0])
    builds.sort()
    searches.sort()
    chk = int((counts.to(torch.int64) * weights).sum().item())
    return {"s": s, "beta": beta, "policy": policy, "build_ms": builds[len(builds) // 2],
            "search_ms": searches[len(searches) // 2], "depth": st["depth"], "root_b": st["root_b"],
            "nodes": st["nodes"], "leaves": st["leaves"], "halvings": st["halvings"], "tests": st["tests"],
            "staged": st["staged"], "total_pairs": st["total_pairs"], "count_checksum": chk}


rows = []
t0 = time.time()
if args.plane:  # k = 2 policies (R23) against the 3-D ones on a planar set
    for pol in ("btree", "octree", "btree2d", "quadtree"):
        for s in (16, 64):
            rows.append(run(s, 0.5, pol))
else:
    for s in (8, 16, 32, 64, 128, 256):
        rows.append(run(s, 0.5, "btree"))
    for beta in (0.1, 0.25, 0.75, 1.0):
        rows.append(run(64, beta, "btree"))
    for s in (8, 32, 64):
        rows.append(run(s, 0.5, "octree"))
    if n <= 4_000_000:  # k = 2 trees on 3-D data: columns through z (at cfg 5 the walk arena exceeds HBM)
        rows.append(run(64, 0.5, "btree2d"))
        rows.append(run(64, 0.5, "quadtree"))
ref = rows[0]["count_checksum"]
for r in rows:
    r["same_counts_as_first"] = r["count_checksum"] == ref
out = {"config": "plane" if args.plane else args.config, "n": n, "reps": args.reps, "device": torch.cuda.get_device_name(0),
       "wall_s": time.time() - t0, "rows": rows}
text = json.dumps(out, indent=1)
print(text)
if args.out:
    with open(args.out, "w") as f:
        f.write(text + "\n")
bad = [r for r in rows if not r["same_counts_as_first"]]
if bad:
    raise SystemExit(f"neighbor counts differ between settings: {bad}")
