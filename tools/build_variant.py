"""Build an A/B variant of the library with extra nvcc flags into
paper_1910_02639_b200/libbtree_<name>.so (timed by tools/gpu_variants.sh via
BT_LIB).  Measurement tooling only.

  python tools/build_variant.py b6 -DBT_WALK_MIN_BLOCKS=6
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1910_02639_b200 import _build  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
out = os.path.join(_build.PKG, f"libbtree_{name}.so")
cmd = [os.environ.get("NVCC", "nvcc"), *_build.NVCC_FLAGS, *flags, *_build.SOURCES, "-o", out]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr[-3000:])
print(out)
