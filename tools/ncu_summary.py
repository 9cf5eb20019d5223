"""Summarise ncu outputs into profiles/: per-kernel launch times (launch list
CSV) and, for a --set full report, the headline metrics + DRAM bytes per launch.

  python tools/ncu_summary.py launches <launches.csv> <out.txt>
  python tools/ncu_summary.py full <report.ncu-rep> <out.txt> [<traffic.json> <kernel-key> <config>]
  python tools/ncu_summary.py headline <out.txt> <traffic.json>
"""
import csv
import json
import subprocess
import sys
from collections import defaultdict


def to_ms(v, unit):
    v = float(str(v).replace(",", ""))
    return {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
            "second": 1e3, "s": 1e3}.get(unit, 1e-6) * v


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = defaultdict(lambda: defaultdict(float))
    order = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (d["ID"], d["Kernel Name"])
        if key not in order:
            order.append(key)
        m = d["Metric Name"]
        if m == "gpu__time_duration.sum":
            per[key]["ms"] = to_ms(d["Metric Value"], d["Metric Unit"])
        elif m.startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(d["Metric Unit"], 1)
            per[key][m] = float(d["Metric Value"].replace(",", "")) * scale
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for key in order:
        name = key[1].split("(")[0].replace("bt::<unnamed>::", "").replace("(anonymous namespace)::", "")
        name = name.split("::")[-1]
        a = agg[name]
        a[0] += 1
        a[1] += per[key].get("ms", 0.0)
        a[2] += per[key].get("dram__bytes_read.sum", 0.0) + per[key].get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values()) or 1.0
    lines = [f"ncu launch list ({len(order)} launches, serialised, cold-cache): {path}",
             f"{'kernel':40s} {'launches':>8s} {'ms':>10s} {'share':>7s} {'DRAM GB':>9s}"]
    for name, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{name:40s} {a[0]:8d} {a[1]:10.3f} {100 * a[1] / tot:6.1f}% {a[2] / 1e9:9.3f}")
    lines.append(f"{'total':40s} {len(order):8d} {tot:10.3f}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep, out, traffic=None, key=None, config=None):
    res = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(res.splitlines()))
    hdr = rows[0]
    want = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
            "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy",
            "Theoretical Occupancy", "Registers Per Thread", "Warp Cycles Per Issued Instruction"]
    lines = [f"ncu --set full summary: {rep}"]
    kernels = defaultdict(list)
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") in want:
            kernels[(d["ID"], d["Kernel Name"][:60])].append(f"{d['Metric Name']}: {d['Metric Value']} {d['Metric Unit']}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    h2 = rr[0]
    dram = {}
    pipes = {}
    for r in rr[2:]:
        d = dict(zip(h2, r))
        # execution pipes at >= 10 % of their sustained peak (XU = POPC / conversions, quarter rate)
        pp = []
        for name, val in d.items():
            if name.startswith("sm__inst_executed_pipe_") and name.endswith(".avg.pct_of_peak_sustained_active"):
                try:
                    v = float(val.replace(",", ""))
                except ValueError:
                    continue
                if v >= 10.0:
                    pp.append((v, name[len("sm__inst_executed_pipe_"):-len(".avg.pct_of_peak_sustained_active")]))
        pipes[(d.get("ID"), d.get("Kernel Name", "")[:60])] = ", ".join(f"{n} {v:.1f} %" for v, n in sorted(pp, reverse=True))
        try:
            rd = float(d.get("dram__bytes_read.sum", "0").replace(",", ""))
            wr = float(d.get("dram__bytes_write.sum", "0").replace(",", ""))
        except ValueError:
            continue
        unit_r = rr[1][h2.index("dram__bytes_read.sum")] if "dram__bytes_read.sum" in h2 else "byte"
        unit_w = rr[1][h2.index("dram__bytes_write.sum")] if "dram__bytes_write.sum" in h2 else "byte"
        sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        dram[(d["ID"], d["Kernel Name"][:60])] = rd * sc.get(unit_r, 1) + wr * sc.get(unit_w, 1)
    for k, v in kernels.items():
        lines.append(f"[{k[0]}] {k[1]}")
        lines += ["    " + x for x in v]
        if k in dram:
            lines.append(f"    dram bytes (read + write): {dram[k]:.4g}")
        if pipes.get(k):
            lines.append(f"    pipes (inst executed, % of sustained peak while active): {pipes[k]}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic and dram:
        t = {}
        try:
            t = json.load(open(traffic))
        except Exception:
            pass
        t.setdefault("kernels", {})
        # bench.py's kernel keys -> the report's kernel of that name (first launch)
        names = {"walk_desc": "desc_kernel", "walk_test": "walk_kernel", "walk_fill": "fill_kernel"}
        for bk, kn in names.items():
            hit = [v for (i, name), v in sorted(dram.items(), key=lambda kv: int(kv[0][0])) if kn in name]
            if hit and (key in (None, "all") or key == bk):
                t["kernels"][bk] = hit[0]
        t["config"] = int(config)
        t["source"] = f"ncu --set full dram__bytes_read.sum + dram__bytes_write.sum ({rep.split('/')[-1]})"
        json.dump(t, open(traffic, "w"), indent=1)


def headline(summary, traffic):
    """The "ncu" block of dram_traffic.json (bench.py's roofline.ncu) from a `full` summary file."""
    import re
    t = json.load(open(traffic))
    out, cur = {}, None
    for line in open(summary):
        m = re.match(r"\[\d+\] .*?(desc_kernel|walk_kernel|fill_kernel)", line)
        if m:
            cur = out.setdefault(m.group(1), {}) if m.group(1) not in out else None
            continue
        if cur is None or not line.startswith("    "):
            continue
        k, _, v = line.strip().partition(": ")
        if k.startswith("pipes"):
            cur["pipes_pct"] = {p.split()[0]: float(p.split()[1]) for p in v.split(", ")}
            continue
        num = re.match(r"([\d.,e+]+)\s*(\S*)", v)
        if not num:
            continue
        x, unit = float(num.group(1).replace(",", "")), num.group(2)
        if k == "Duration":
            cur["duration_ms"] = x * {"us": 1e-3, "ms": 1.0, "s": 1e3}.get(unit, 1.0)
        elif k == "L2 Hit Rate":
            cur["l2_hit_pct"] = x
        elif k == "Issue Slots Busy":
            cur["issue_slots_busy_pct"] = x
        elif k == "Executed Ipc Active":
            cur["ipc"] = x
        elif k == "Achieved Occupancy":
            cur["occupancy_pct"] = x
        elif k.startswith("dram bytes"):
            cur["dram_bytes"] = x
    for d in out.values():
        if "dram_bytes" in d and d.get("duration_ms"):
            d["dram_GBps"] = d["dram_bytes"] / d["duration_ms"] / 1e6
    out["source"] = summary
    t["ncu"] = out
    json.dump(t, open(traffic, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "headline":
        headline(sys.argv[2], sys.argv[3])
    elif sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(*sys.argv[2:])
