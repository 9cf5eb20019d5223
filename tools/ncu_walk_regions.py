"""walk_kernel instruction / stall-sample shares by code region, plus the top
source lines of the walk, fill and descent kernels, from an ncu --set full
report captured with --import-source on (lines of walk.cu at capture time).

  ncu -i rep --page source --csv --print-source cuda,sass > src.csv
  python tools/ncu_walk_regions.py src.csv
"""
import csv
import re
import sys

WALK = "paper_1910_02639_b200/csrc/walk.cu"


def regions_from_source():
    """Line ranges of the walk kernel's code regions, found by their anchors."""
    lines = open(WALK).read().split("\n")

    def at(pat):
        for i, l in enumerate(lines, 1):
            if re.search(pat, l):
                return i
        raise SystemExit(f"anchor not found: {pat}")
    a = {k: at(p) for k, p in {
        "helpers": r"double warp_min\(double v\)", "unit_setup": r"void unit_setup\(",
        "claims": r"^struct WorkBatch", "desc": r"^struct DescOut", "resolve": r"void resolve_band\(",
        "test_pre": r"int2 test_block\(", "test_loop": r"^    float4 N0, N1;", "test_post": r"const bool band = S.u.force",
        "locate": r"void locate\(", "stage": r"void stage_group\(", "kernel": r"walk_kernel\(WalkArgs a\)",
        "k_stage": r"// ---- staging phase", "k_test": r"// ---- test phase", "k_epi": r"const int nstaged = slot0;",
        "fill": r"^// Fill pass"}.items()}
    return [("helpers (packed-fp32 / vote wrappers)", a["helpers"], a["unit_setup"] - 1),
            ("unit_setup", a["unit_setup"], a["claims"] - 1), ("work claims / slabs", a["claims"], a["desc"] - 1),
            ("resolve_band (exact fp64 band)", a["resolve"], a["test_pre"] - 1),
            ("test_block prologue", a["test_pre"], a["test_loop"] - 1),
            ("test_loop (f32x2 pair tests + ballots)", a["test_loop"], a["test_post"] - 1),
            ("test_block epilogue (self, counts, mask record)", a["test_post"], a["locate"] - 1),
            ("locate", a["locate"], a["stage"] - 1), ("stage_group (load, cull, scratch)", a["stage"], a["kernel"] - 1),
            ("walk_kernel unit setup", a["kernel"], a["k_stage"] - 1),
            ("walk_kernel staging driver", a["k_stage"], a["k_test"] - 1),
            ("walk_kernel test driver", a["k_test"], a["k_epi"] - 1),
            ("walk_kernel epilogue", a["k_epi"], a["fill"] - 1)]


def main(path, regions):
    rows = list(csv.reader(open(path)))
    blocks, cur, fpath = [], None, "?"
    for r in rows:
        if r and r[0] == "Function Name":
            cur = [r[1], None, []]
            blocks.append(cur)
        elif r and r[0] == "File Path":
            fpath = r[1]
        elif r and r[0] == "Line No" and cur is not None:
            cur[1] = r
        elif cur and cur[1] and r and r[0].isdigit():
            cur[2].append((fpath.split("/")[-1], r))

    def agg(sub):
        out = []
        for name, hdr, d in blocks:
            if sub not in name:
                continue
            ii, si = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
            for f, r in d:
                try:
                    out.append((f, int(r[0]), float(r[ii] or 0), float(r[si] or 0), r[1][:90]))
                except ValueError:
                    pass
        return out
    w = agg("walk_kernel")
    tot, tots = sum(x[2] for x in w) or 1, sum(x[3] for x in w) or 1
    print("walk_kernel<0> instruction / stall-sample shares by code region (walk.cu at capture time):")
    print(f"total instructions {tot:.4g}, stall samples {int(tots)}")
    R = {n: [0.0, 0.0] for n, _, _ in regions}
    other = [0.0, 0.0]
    for f, ln, a, b, _ in w:
        for n, lo, hi in regions:
            if f == "walk.cu" and lo <= ln <= hi:
                R[n][0] += a
                R[n][1] += b
                break
        else:
            other[0] += a
            other[1] += b
    for n, v in sorted(R.items(), key=lambda kv: -kv[1][0]):
        print(f"  {n:50s} instr {100 * v[0] / tot:5.1f}%   stall samples {100 * v[1] / tots:5.1f}%")
    print(f"  {'other (CUDA headers: ballot / shuffle intrinsics)':50s} instr {100 * other[0] / tot:5.1f}%   "
          f"stall samples {100 * other[1] / tots:5.1f}%")
    for k in ("walk_kernel", "fill_kernel", "desc_kernel"):
        d = agg(k)
        t, ts = sum(x[2] for x in d) or 1, sum(x[3] for x in d) or 1
        print(f"\n{k} top source lines by stall samples (total instr {t:.4g}):")
        for f, ln, a, b, src in sorted(d, key=lambda x: -x[3])[:12]:
            print(f"  {100 * b / ts:5.1f}% smp {100 * a / t:5.1f}% ins {f}:{ln}: {src}")


if __name__ == "__main__":
    main(sys.argv[1], regions_from_source())
