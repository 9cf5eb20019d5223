"""bench.py -- b-tree exact close-neighbor search on B200 (arXiv 1910.02639).

One step = one pass of the whole hot path over one particle set resident in
HBM: bt_build (root box, levels of Eq. 1-4 + scatter, leaves) +
bt_find_neighbors (count pass, offsets scan, capacity check, fill pass into
the CSR) + bt_free.  Workload: BASELINE.json configs[4] ("cfg 5",
N = 2^25, ngmax = 512, count-then-fill CSR), seeded synthetic data.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl b200|reference]

Multi-GPU (torchrun): every rank searches its own independently drawn
sub-domain of the same recipe (the paper's per-node sub-domain);
no data-path collective; weak scaling; time = max over ranks.
--mode replicated: one particle set of the cfg size for the whole job (SURVEY
8(e) variant (i)): each step rank 0 broadcasts pos and h (NCCL), every rank
builds the same tree and searches only its share of the work units
(bt_set_partition); strong scaling.
--impl reference runs the CPU oracle (oracle/, the paper's Alg. 1 + Alg. 2 in
plain C) on a bounded sample, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_1910_02639_b200 import datagen  # noqa: E402

WORKLOADS = {
    1: "N=10,000 uniform [0,1)^3, h=0.0668, s=64",
    2: "N=1,000,000 uniform [0,1)^3, h_i=0.0144*U(0.8,1.2), s=64",
    3: "100^3 jittered lattice, h=0.015, s=64",
    4: "N=4,000,000 Evrard-like sphere, h from n(r), s=64",
    5: "N=33,554,432: 50% uniform + 50% in 64 Gaussian clumps (sigma 0.01), h from a 64^3 histogram, "
       "s=64, max_empty=0.5, ngmax=512, count-then-fill CSR",
}
METRIC = "neighbor-search particles/s (build + count + fill, all particles)"
UNIT = "particles/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--n", type=int, default=None, help="override particle count (not a bench line)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--mode", default="subdomain", choices=["subdomain", "replicated"],
                    help="subdomain: one sub-domain per rank (weak); replicated: one set, units sharded (strong)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tree-order", action="store_true",
                    help="skip the secondary tree-order measurement (bt_set_tree_order, P:491)")
    ap.add_argument("--cpu-sample", type=int, default=None,
                    help="oracle queries timed for cpu_baseline (default: every query up to N = 4.2M, else 1M)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank time over all ranks (identity without a process group)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def subdomain(cfg: int, n, rank: int):
    """Rank r's own sub-domain: the cfg recipe drawn with seed offset r (weak scaling)."""
    return datagen.make_config(cfg, n=n, seed_offset=rank)


def replicated_inputs(cfg: int, n, rank: int, device):
    """--mode replicated: rank 0 draws the job's one particle set; the other
    ranks allocate buffers that the per-step broadcast fills."""
    import torch
    if rank == 0:
        pos_np, h_np = subdomain(cfg, n, 0)
        return pos_np, h_np, torch.from_numpy(pos_np).to(device), torch.from_numpy(h_np).to(device)
    nn = n if n is not None else datagen.FULL_N[cfg]
    return (None, None, torch.empty((nn, 3), dtype=torch.float64, device=device),
            torch.empty(nn, dtype=torch.float64, device=device))


def broadcast_inputs(pos, h):
    """The step's particle set from rank 0 to every rank (NCCL over NVLink on the GPUs)."""
    import torch.distributed as dist
    dist.broadcast(pos, 0)
    dist.broadcast(h, 0)


def strong_value(n_total: int, ms: float) -> float:
    """Whole-job throughput of one shared particle set over the max-over-ranks step time."""
    return n_total / (ms * 1e-3)


def weak_value(n_per_rank: int, ws: int, ms: float) -> float:
    """Whole-job throughput: all ranks' particles over the max-over-ranks step time."""
    return n_per_rank * ws / (ms * 1e-3)


def config_block(cfg, n, ws, mode="subdomain"):
    nn = n if n is not None else datagen.FULL_N[cfg]
    par = (f"replicas only: {ws} independent sub-domains (one full cfg-size particle set per GPU, no split of one "
           f"set; --mode replicated splits one set)" if mode == "subdomain"
           else f"one particle set split over {ws} GPUs: replicated tree, work units sharded (pos/h broadcast per step)")
    return {"workload": (f"BASELINE.json configs[{cfg - 1}] (cfg {cfg}): {WORKLOADS[cfg]}"
                         + ("" if n is None else f" [n overridden to {n}: not a bench line]")),
            ("N_per_gpu" if mode == "subdomain" else "N_total"): nn, "bucket_size": datagen.BUCKET_SIZE,
            "max_empty": datagen.MAX_EMPTY, "alpha": 0.5, "ngmax": datagen.NGMAX, "parallelism": par,
            "l2": "inputs larger than L2 (pos 805 MB + h 268 MB at cfg 5); no flush"}


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for k, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(k)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU oracle: cpu_baseline / --impl reference
# ---------------------------------------------------------------------------
def cpu_model() -> str:
    """The host CPU's model name (/proc/cpuinfo), for the CPU-baseline line."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def default_sample(n: int) -> int:
    """Oracle queries timed per cpu_baseline: the whole workload up to N = 4.2M
    (cfg 1-4: tens of seconds on the box's cores), a 1M-query sample above."""
    return n if n <= 4_200_000 else 1_000_000


def oracle_sample(pos, h, sample_queries: int):
    """Time the oracle as it stands on this host: full BuildTree + the
    FindNeighbors count and row passes over every query (N <= 4.2M) or a
    random sample of queries, all host cores (OpenMP over queries).  Returns
    (seconds per full step -- measured, or scaled from the sample --,
    description, cores, build s, search s)."""
    import oracle
    n = pos.shape[0]
    cores = oracle.default_threads()
    t0 = time.perf_counter()
    tree = oracle.Tree(pos, datagen.BUCKET_SIZE, datagen.MAX_EMPTY)
    t1 = time.perf_counter()
    k = min(sample_queries, n)
    if k >= n:
        tree.neighbors(h, threads=cores)
    else:
        rng = np.random.default_rng(7)
        q = np.sort(rng.choice(n, k, replace=False)).astype(np.int64)
        tree.neighbors(h, queries=q, threads=cores)
    t2 = time.perf_counter()
    build_s = t1 - t0
    search_s = (t2 - t1) * n / k
    if k >= n:
        desc = (f"oracle on the whole workload, measured: BuildTree on all {n} particles ({build_s:.2f} s, "
                f"1 thread) + count and row passes for all {n} queries ({t2 - t1:.2f} s, {cores} threads); "
                f"host CPU: {cpu_model()}")
    else:
        desc = (f"oracle BuildTree on all {n} particles ({build_s:.2f} s, 1 thread) + count and row passes for "
                f"{k} random queries ({t2 - t1:.2f} s, {cores} threads), search scaled x{n / k:.1f} to all "
                f"queries (full single-thread and all-core runs: profiles/r02_oracle_baseline.jsonl); "
                f"host CPU: {cpu_model()}")
    return build_s + search_s, desc, cores, build_s, search_s


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    pos, h = datagen.make_config(args.config, n=args.n)
    n = pos.shape[0]
    steps, walls = [], []
    desc = cores = None
    k = min(args.cpu_sample or default_sample(n), 200_000) if n > 4_200_000 else default_sample(n)
    for s in range(args.warmup + args.steps):
        w0 = time.perf_counter()
        step_s, desc, cores, b, srch = oracle_sample(pos, h, k)
        if s >= args.warmup:
            steps.append(step_s)
            walls.append(time.perf_counter() - w0)
    t = float(np.mean(steps))
    v = n / t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded numpy PCG64, SURVEY 8(d) recipe)",
            "config": config_block(args.config, args.n, 1),
            # a step times BuildTree on all N and the search of the whole workload (N <= 4.2M) or of k
            # sampled queries; ms_per_step / value scale the sampled search to all N queries
            "sampled": k < n, "ms_per_step_measured_wall": float(np.mean(walls)) * 1e3,
            "full_measured_runs": "profiles/r02_oracle_baseline.jsonl (tools/oracle_baseline.py: every query, "
                                  "1 thread and all cores)",
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def run_b200(args):
    import torch

    import paper_1910_02639_b200 as P

    ws, rank, local = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the product path has no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    P.lib()

    replicated = args.mode == "replicated"
    if replicated:  # rank 0's particle set arrives by broadcast every step
        pos_np, h_np, pos, h = replicated_inputs(args.config, args.n, rank, dev)
    else:
        pos_np, h_np = subdomain(args.config, args.n, rank)
        pos = torch.from_numpy(pos_np).to(dev)
        h = torch.from_numpy(h_np).to(dev)
    n = pos.shape[0]
    ngmax = datagen.NGMAX
    counts = torch.empty(n, dtype=torch.int32, device=dev)
    offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
    nbr = torch.empty(n * ngmax, dtype=torch.int32, device=dev)  # capacity n * ngmax (BJ)
    stream = torch.cuda.current_stream()

    def step():
        if replicated and ws > 1:  # the step's particle set, from rank 0 (NVLink)
            broadcast_inputs(pos, h)
        t = P.Tree(pos, datagen.BUCKET_SIZE, datagen.MAX_EMPTY)
        if replicated:
            t.set_partition(rank, ws)
        t.find_neighbors(h, ngmax, counts=counts, offsets=offsets, nbr_idx=nbr)
        st = t.stats()
        t.free()
        return st

    for _ in range(args.warmup):
        st = step()
    torch.cuda.synchronize()

    P.profile_reset()
    P.profile_enable(True)
    clocks = ClockSampler(local)
    clocks.start()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        st = step()
    e1.record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    clk = clocks.stop()
    P.profile_enable(False)
    prof = P.profile()
    ms = max_over_ranks(ms, dev)
    total_pairs = int(st["total_pairs"])

    def ph(name):
        return prof.get(name, (0.0, 0))[0] / args.steps

    launches = sum(v[1] for k, v in prof.items() if k.startswith("kernel.")) // args.steps
    kern = {"build": ph("build.total"), "walk_desc": ph("search.desc") + ph("search.desc_big"),
            "walk_test": ph("search.count"), "scan": ph("search.scan"), "walk_fill": ph("search.fill"),
            "search_total": ph("search.total")}
    if ph("search.gather_h") > 0:  # (the count call gathers h inside its descent; separate only when partitioned)
        kern["gather_h"] = ph("search.gather_h")

    # ---- roofline of the dominant kernel -----------------
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    loaded, staged, tests = int(st["loaded"]), int(st["staged"]), int(st["tests"])
    dom = max(("walk_desc", "walk_test", "walk_fill", "build"), key=lambda k: kern[k])
    if dom == "walk_test":
        # walk_kernel: staging + pair tests, bound by fp32 issue.  Algorithmic
        # work = the plain predicate's 8 flops per pair test (3 differences, 3
        # squares, 2 sums), against the measured packed-fp32 peak counted the
        # same way: 23.61 T FFMA2 instruction-lanes/s x 2 FMAs x 2 flops =
        # 94.4 TFLOP/s (tools/probe_rates.cu, profiles/r01_probe_rates.txt).
        # (The kernel issues 4 fp32 element ops per pair -- FADD + 3 FFMA of the
        # expanded form -- against 47.2 T element-ops/s: the same fraction.)
        alu_peak = 94.44
        achieved = tests * 8 / (kern[dom] * 1e-3) / 1e12
        roofline = {"kernel": "walk_kernel (A10 staging + A11 pair tests)", "bound": "alu", "achieved": achieved,
                    "peak": alu_peak, "unit": "TFLOP/s", "frac": achieved / alu_peak, "traffic": None,
                    "peak_source": "measured: packed FFMA2 rate x 2 FMA x 2 flops (tools/probe_rates.cu, "
                                   "profiles/r01_probe_rates.txt)",
                    "algorithmic_flops": tests * 8, "issued_fp32_element_ops": tests * 4}
    else:
        if dom == "walk_desc":
            # descent: per unit the query records (32 B) + h (8 B), per listed leaf
            # its box (48 B) + count (4 B) read and its id (4 B) written
            alg_bytes = n * 40 + int(st.get("list_entries", 0)) * 56
        elif dom == "walk_fill":
            # recorded masks (8 B/word) + candidate indices (4 B/slot) read, per
            # particle record + offset read, 4-B output index per neighbor pair
            alg_bytes = int(st["mask_words"]) * 8 + staged * 4 + n * (32 + 8) + 4 * total_pairs
        else:
            # build: per particle pos read (24 B) + records written / re-read over
            # the levels and the final sort (~4 x 32 B)
            alg_bytes = n * (24 + 4 * 32)
        achieved = alg_bytes / (kern[dom] * 1e-3) / 1e9
        roofline = {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                    "frac": achieved / hbm_peak, "traffic": None, "peak_source": hbm_src,
                    "algorithmic_bytes": alg_bytes}
    try:  # per-launch DRAM bytes / L2 hit rate from the committed ncu captures (profiles/), if any
        tr = json.load(open(os.path.join(ROOT, "profiles", "dram_traffic.json")))
        if tr.get("config") == args.config and dom in tr.get("kernels", {}):
            roofline["traffic"] = tr["kernels"][dom]
            roofline["traffic_source"] = tr.get("source")
        if tr.get("config") == args.config and tr.get("ncu"):
            roofline["ncu"] = tr["ncu"]
    except Exception:
        pass
    # BASELINE.json's own definition: bytes of candidate positions actually read
    # by the walk (16-B compact records loaded by the staging) over the time of
    # the whole bt_find_neighbors call (gather of h, descent, count, offsets
    # scan, capacity check, fill) and peak HBM bandwidth
    bcand = loaded * 16
    search_ms = ph("search.total")
    bj_roof = {"B_cand_bytes": bcand, "search_ms": search_ms,
               "frac": (bcand / (search_ms * 1e-3) / 1e9) / hbm_peak if search_ms > 0 else None,
               "definition": "16 B x compact records loaded by the walk staging / whole bt_find_neighbors time / "
                             "measured HBM peak"}

    # ---- secondary: the same step in the tree-order index space ---------------
    # (bt_set_tree_order: particles reordered along the walk's curve; the
    # step gathers h into tree order with bt_reorder, then count + fill write
    # rows and neighbor indices by tree position -- the rows of one work unit
    # are one contiguous range of the CSR)
    tree_order = None
    if not replicated and not args.no_tree_order and args.steps > 0:
        h_t = torch.empty_like(h)

        def step_to():
            t = P.Tree(pos, datagen.BUCKET_SIZE, datagen.MAX_EMPTY)
            t.set_tree_order(True)
            t.reorder(h, out=h_t)
            t.find_neighbors(h_t, ngmax, counts=counts, offsets=offsets, nbr_idx=nbr)
            s2 = t.stats()
            t.free()
            return s2

        step_to()
        P.profile_reset()
        P.profile_enable(True)
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            s2 = step_to()
        g1.record(stream)
        torch.cuda.synchronize()
        P.profile_enable(False)
        prof2 = P.profile()
        tms = max_over_ranks(g0.elapsed_time(g1) / args.steps, dev)

        def ph2(name):
            return prof2.get(name, (0.0, 0))[0] / args.steps

        assert int(s2["total_pairs"]) == total_pairs
        tree_order = {"value": weak_value(n, ws, tms), "unit": UNIT, "ms_per_step": tms,
                      "kernel_ms": {"build": ph2("build.total"), "walk_desc": ph2("search.desc"),
                                    "walk_test": ph2("search.count"), "walk_fill": ph2("search.fill"),
                                    "search_total": ph2("search.total")},
                      "api": "bt_set_tree_order + bt_reorder(h) + bt_find_neighbors (rows and indices by tree "
                             "position; same pairs)"}

    # ---- end to end through the public API on host buffers --------------------
    e2e = None
    if replicated:
        e2e = {"value": None, "note": "not measured in --mode replicated (bt_search_host searches the whole set)"}
    elif not args.no_e2e and args.e2e_steps > 0:
        pos_h = torch.from_numpy(pos_np).pin_memory()
        h_h = torch.from_numpy(h_np).pin_memory()
        c_h = torch.empty(n, dtype=torch.int32).pin_memory()
        o_h = torch.empty(n + 1, dtype=torch.int64).pin_memory()
        nb_h = torch.empty(max(total_pairs, 1), dtype=torch.int32).pin_memory()
        del nbr
        torch.cuda.empty_cache()
        P.search_host(pos_h, h_h, capacity=total_pairs, counts=c_h, offsets=o_h, nbr=nb_h)  # warm-up
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.e2e_steps):
            P.search_host(pos_h, h_h, capacity=total_pairs, counts=c_h, offsets=o_h, nbr=nb_h)
        f1.record(stream)
        torch.cuda.synchronize()
        ems = f0.elapsed_time(f1) / args.e2e_steps
        ems = max_over_ranks(ems, dev)
        e2e = {"value": weak_value(n, ws, ems), "unit": UNIT, "ms_per_step": ems,
               "h2d_bytes_per_step": n * 32, "d2h_bytes_per_step": n * 4 + (n + 1) * 8 + 4 * total_pairs,
               "api": "bt_search_host (pinned host buffers; H2D pos+h, build, count, fill, D2H counts+offsets+CSR)"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        step_s, desc, cores, _, _ = oracle_sample(pos_np, h_np, args.cpu_sample or default_sample(n))
        cpu = {"value": n / step_s, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}

    if rank == 0:
        value = strong_value(n, ms) if replicated else weak_value(n, ws, ms)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong" if replicated else "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded numpy PCG64, SURVEY 8(d) recipe)",
                "config": config_block(args.config, args.n, ws, args.mode),
                "pairs_per_s": (None if replicated else total_pairs * ws / (ms * 1e-3)),
                ("total_pairs_rank0" if replicated else "total_pairs_per_gpu"): total_pairs,
                "build_ms": kern["build"], "kernel_ms": kern, "gpu_launches": launches,
                "roofline": roofline, "bj_hbm_roofline": bj_roof,
                "tree": {k: st[k] for k in ("depth", "root_b", "nodes", "leaves", "halvings", "units")},
                "walk_counters": {k: st.get(k) for k in ("loaded", "staged", "tests", "exact_tests", "mask_words",
                                                         "cand_slots", "list_entries", "big_units", "mask_words_nonzero")},
                "tree_order": tree_order, "clocks": clk, "e2e": e2e, "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
