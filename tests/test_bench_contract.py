"""CPU checks of bench.py's JSON contract: the --impl reference leg (the CPU
oracle, the one bench path that runs without a GPU) prints one JSON line with
the keys the driver reads, and the host-side helpers compute the documented
whole-job values."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_leg_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--n", "20000",
                          "--steps", "2", "--warmup", "1", "--cpu-sample", "5000"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 1
    assert d["value"] > 0 and d["higher_is_better"] is True and d["unit"] == "particles/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["value"] == pytest.approx(20000 / (d["ms_per_step"] * 1e-3))
    assert "workload" in d["config"] and "cfg 5" in d["config"]["workload"]


def test_value_helpers():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.weak_value(1000, 4, 2.0) == pytest.approx(4000 / 2e-3)
    assert bench.strong_value(1000, 2.0) == pytest.approx(1000 / 2e-3)
    c = bench.config_block(5, None, 2)
    assert c["N_per_gpu"] == 2 ** 25 and "replicas only: 2 independent sub-domains" in c["parallelism"]
    r = bench.config_block(5, None, 8, "replicated")
    assert r["N_total"] == 2 ** 25 and "replicated" in r["parallelism"]
