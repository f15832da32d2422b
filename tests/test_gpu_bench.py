"""bench.py end to end on the GPU at a small size: one JSON line with every contract key, clean bin counts
(each set counted once), and the verdict-only / device-generation / DES legs present."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_small_run_contract():
    cmd = [sys.executable, "bench.py", "--sets-per-gpu", "20000", "--steps", "3", "--warmup", "3",
           "--des-sets", "2000", "--des-horizon-s", "1", "--cpu-budget", "1"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "config", "gpu_launches", "clocks", "roofline", "e2e", "cpu_baseline", "verdict_only",
              "e2e_device_generate", "des", "bins"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert sum(d["bins"][0::2]) == 20000
    assert 0 < sum(d["bins"][1::2]) < 20000
    assert d["gpu_launches"] >= 3  # one fused_kernel launch per step (device-resident batch)
    assert d["des"]["sim_le_bound_violations"] == 0
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["verdict_only"]["value"] > 0 and d["e2e_device_generate"]["value"] > 0
