"""Time bt_density (neighbor search fused with the SPH density sum) against
count + fill at one configuration, and report its error against the oracle on
sampled rows (tolerance derivation: DESIGN.md section 11c)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1910_02639_b200 as P  # noqa: E402
from paper_1910_02639_b200 import datagen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--sample", type=int, default=20000)
args = ap.parse_args()

pos_np, h_np = datagen.make_config(args.config, n=args.n)
n = pos_np.shape[0]
m_np = np.random.default_rng(11).uniform(0.5, 1.5, n)
dev = torch.device("cuda:0")
pos, h, m = (torch.from_numpy(x).to(dev) for x in (pos_np, h_np, m_np))
t = P.build(pos)
counts = torch.empty(n, dtype=torch.int32, device=dev)
offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
nbr = torch.empty(n * 512, dtype=torch.int32, device=dev)
res = {}
for name, fn in (("density", lambda: t.density(h, m)),
                 ("count_fill", lambda: t.find_neighbors(h, 512, counts=counts, offsets=offsets, nbr_idx=nbr))):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    res[name + "_ms"] = e0.elapsed_time(e1) / args.reps
rho = t.density(h, m).cpu().numpy()
q = np.sort(np.random.default_rng(2).choice(n, min(args.sample, n), replace=False)).astype(np.int64)
ref = oracle.Tree(pos_np, 64, 0.5).density(h_np, m_np, queries=q)
rel = np.abs(rho[q] - ref) / ref
res.update({"config": args.config, "n": n, "sampled_rows": int(q.size), "max_rel_err": float(rel.max()),
            "p99_rel_err": float(np.quantile(rel, 0.99)), "mean_rel_err": float(rel.mean()),
            "density_particles_per_s": n / (res["density_ms"] * 1e-3)})
print(json.dumps(res, indent=1))
