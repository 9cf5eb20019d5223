"""Full (non-extrapolated) CPU-oracle baseline per BASELINE.json config, on
the host it runs on (run it on the GPU box: `gpurun -- python
tools/oracle_baseline.py ...`).  Times the oracle as it stands (oracle/: the
paper's Alg. 1 build and Alg. 2 walk in plain C, count pass + row pass over
every query) single-threaded and on all host cores, and prints one JSON line
per config.  Test/measurement infrastructure: the product never runs it.

  python tools/oracle_baseline.py --configs 1 2 3 4 5 [--single 1 2 3 4 5] [--reps 3]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1910_02639_b200 import datagen  # noqa: E402


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[1, 2, 3, 4, 5])
    ap.add_argument("--single", type=int, nargs="*", default=[1, 2, 3, 4],
                    help="configs whose full search is also timed on one thread")
    ap.add_argument("--reps", type=int, default=1)
    args = ap.parse_args()
    cores = oracle.default_threads()
    for cfg in args.configs:
        pos, h = datagen.make_config(cfg)
        n = pos.shape[0]
        builds, alls, ones = [], [], []
        pairs = None
        for _ in range(args.reps):
            t0 = time.perf_counter()
            tree = oracle.Tree(pos, datagen.BUCKET_SIZE, datagen.MAX_EMPTY)
            t1 = time.perf_counter()
            c, off, _ = tree.neighbors(h, threads=cores)
            t2 = time.perf_counter()
            builds.append(t1 - t0)
            alls.append(t2 - t1)
            pairs = int(off[-1])
            del c, off
            if cfg in args.single:
                t3 = time.perf_counter()
                tree.neighbors(h, threads=1)
                ones.append(time.perf_counter() - t3)
            del tree
        b = float(np.median(builds))
        sa = float(np.median(alls))
        s1 = float(np.median(ones)) if ones else None
        print(json.dumps({
            "config": cfg, "n": n, "total_pairs": pairs, "host_cores": cores, "host_cpu": cpu_model(),
            "what": "oracle/ as it stands: BuildTree (Alg. 1, one thread) + count pass and row pass of "
                    "FindNeighbors (Alg. 2) over every query (OpenMP over queries); full workload, no sampling",
            "reps": args.reps, "build_s": b, "search_s_all_cores": sa, "search_s_1_thread": s1,
            "particles_per_s_all_cores": n / (b + sa), "pairs_per_s_all_cores": pairs / sa,
            "particles_per_s_1_thread": (n / (b + s1)) if s1 else None,
            "search_particles_per_s_all_cores": n / sa}), flush=True)


if __name__ == "__main__":
    main()
