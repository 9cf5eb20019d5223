"""The C ABI from plain C: examples/c_search.c compiles and links against
libbtree.so and the CUDA runtime here (no GPU needed); on a B200 it runs the
host-buffer and device-pointer paths and checks sampled counts against a
direct double loop with the same predicate."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = "/usr/local/cuda"


def _compile(out):
    import paper_1910_02639_b200 as P
    P.lib()  # builds libbtree.so if needed
    pkg = os.path.join(ROOT, "paper_1910_02639_b200")
    cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", os.path.join(ROOT, "examples", "c_search.c"),
           "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(CUDA, "include"), "-L" + pkg, "-lbtree",
           "-L" + os.path.join(CUDA, "lib64"), "-lcudart", "-Wl,-rpath," + pkg, "-o", out]
    subprocess.check_call(cmd)


def test_c_example_builds(tmp_path):
    if not os.path.exists(os.path.join(CUDA, "include", "cuda_runtime.h")):
        pytest.skip("no CUDA toolkit headers")
    out = str(tmp_path / "c_search")
    _compile(out)
    assert os.path.exists(out)


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = str(tmp_path / "c_search")
    _compile(out)
    r = subprocess.run([out, "100000"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "c_search ok" in r.stdout
