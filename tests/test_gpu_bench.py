"""bench.py's JSON contract on the GPU (small config C1 so it runs in seconds): one line
with the driver's keys, a roofline object, the clock sample, the e2e object and a
positive launch count; and the reference arm's line."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_line_contract_c1():
    d = _run("--config", "C1", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-ttt")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "e2e", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert d["dtype"] == "f64" and "workload" in d["config"]
    assert d["gpu_launches"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


def test_bench_reference_arm_line():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "1", "--cpu-m", "5000", "--cpu-n", "1000")
    assert d["impl"] == "reference"
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_bench_block_placement_small():
    # the block-major data path (datagen.generate_blocks, placement.plan) on one GPU:
    # configs[3]'s softmax with 8 feature blocks at a small size
    d = _run("--config", "C4", "--m", "4000", "--n", "2048", "--kappa", "40", "--steps", "3", "--warmup", "3",
             "--no-cpu", "--no-ttt")
    assert d["config"]["placement"].startswith("block-major") and d["config"]["local_blocks"] == 8
    assert d["scaling"] == "strong" and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["value"] > 0

