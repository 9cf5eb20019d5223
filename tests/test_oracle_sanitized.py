"""The oracle under AddressSanitizer + UndefinedBehaviorSanitizer (SURVEY
section 5): the same C source compiled with -fsanitize=address,undefined,
loaded in a child interpreter, runs every entry point on small cases (tree
build for the four policies, walk, brute force, symmetric brute force,
density).  Any invalid access or undefined behaviour aborts the child."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import numpy as np, oracle
from paper_1910_02639_b200 import datagen
pos, h = datagen.clustered(3000, 5, h=0.02)
h = h * np.random.default_rng(6).uniform(0.5, 2.0, len(h))
for pol in ("btree", "octree", "btree2d", "quadtree"):
    for s in (1, 8, 64):
        t = oracle.Tree(pos, s, 0.5, policy=pol)
        c, o, i = t.neighbors(h)
        t.order(); t.stats(); t.density(h, np.ones_like(h))
b = oracle.brute_force(pos, h)
bs = oracle.brute_force(pos, h, symmetric=True)
bd = oracle.brute_density(pos, h, np.ones_like(h))
oracle.Tree(np.zeros((0, 3)), 8).stats()
oracle.Tree(np.tile([[0.5, 0.5, 0.5]], (40, 1)), 8, depth_cap=64).neighbors(np.full(40, 0.1))
print("sanitized ok", int(c.sum()), int(bs[0].sum()))
'''


def test_oracle_under_asan_ubsan(tmp_path):
    asan = subprocess.run(["gcc", "-print-file-name=libasan.so"], capture_output=True, text=True).stdout.strip()
    if not asan or not os.path.isabs(asan) or not os.path.exists(asan):
        pytest.skip("no libasan")
    sys.path.insert(0, ROOT)
    import oracle
    lib = tmp_path / "liboracle_asan.so"
    cmd = ["gcc", *oracle.CFLAGS, "-fsanitize=address,undefined", "-fno-omit-frame-pointer",
           "-fno-sanitize-recover=all", os.path.join(ROOT, "oracle", "btree_oracle.c"), "-o", str(lib), "-lm"]
    subprocess.check_call(cmd)
    env = dict(os.environ, ORACLE_LIB=str(lib), LD_PRELOAD=asan, ASAN_OPTIONS="detect_leaks=0:abort_on_error=1",
               UBSAN_OPTIONS="halt_on_error=1:print_stacktrace=1", OMP_NUM_THREADS="2", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", SCRIPT], capture_output=True, text=True, env=env, cwd=ROOT,
                       timeout=600)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-4000:])
    assert "sanitized ok" in r.stdout
