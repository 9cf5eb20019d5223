"""Measurement probe: time writing the cfg 5 CSR (real offsets, tree-order vs
caller-order row visits) with a plain warp-per-row kernel, next to the fill."""
import ctypes as C
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1910_02639_b200 as P  # noqa: E402
from paper_1910_02639_b200 import datagen  # noqa: E402

so = os.path.join(ROOT, "tools", "probe_csr.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                       os.path.join(ROOT, "tools", "probe_csr.cu"), "-o", so])
L = C.CDLL(so)
L.probe_rows.restype = C.c_float
L.probe_rows.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int, C.c_int]
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
pos, h = datagen.make_config(cfg)
dev = torch.device("cuda:0")
pos = torch.from_numpy(pos).to(dev)
h = torch.from_numpy(h).to(dev)
t = P.Tree(pos, 64, 0.5)
counts, offsets = t.count(h)
perm, _, _, _ = t.order()
total = int(offsets[-1])
nbr = torch.empty(total, dtype=torch.int32, device=dev)
res = {"config": cfg, "pairs": total, "bytes": total * 4}
for mode, name in ((0, "tree_order_rows"), (1, "caller_order_rows"), (2, "tree_order_rows_batched_bounds")):
    ms = L.probe_rows(offsets.data_ptr(), perm.data_ptr(), pos.shape[0], nbr.data_ptr(), mode, 5)
    res[name + "_ms"] = ms
    res[name + "_GBps"] = total * 4 / ms / 1e6
P.profile_reset()
P.profile_enable(True)
t.fill(h, offsets, out=nbr)
torch.cuda.synchronize()
res["fill_ms"] = P.profile().get("search.fill", (0, 0))[0]
print(json.dumps(res))
