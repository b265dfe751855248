"""bench.py on the GPU (the driver's round-end step, short): one JSON line with the contract's keys -- the
headline value over two batches in flight, the one-at-a-time latency, e2e with its copy sizes, the roofline of
K1 and the clocks -- and the pipelined and sequential runs agree on every count (bench.py checks that itself)."""
import json
import subprocess
import sys

import pytest

from .conftest import REPO

pytestmark = pytest.mark.gpu


def test_bench_line_contract():
    r = subprocess.run([sys.executable, str(REPO / "bench.py"), "--steps", "3", "--warmup", "3", "--quick",
                        "--no-cpu-baseline"], capture_output=True, text=True, timeout=900, cwd=REPO)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "gpu_launches", "clocks", "pipelining"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] >= 3
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 1000 * 3 * 16 * 11 * 8
    assert d["e2e"]["d2h_bytes_per_step"] > d["e2e"]["h2d_bytes_per_step"]
    assert d["gpu_launches"] >= 3                       # start score, order, K1, verdict
    rf = d["roofline"]
    assert 0 < rf["frac"] <= 1 and rf["unit"] == "TFLOP/s" and rf["kernel_ms"] > 0
    assert d["pipelining"]["batch_latency_ms"] >= d["ms_per_step"] * 0.9   # two in flight: not slower per batch
    assert abs(d["feasible_fraction"] - 0.765) < 1e-9   # the headline batch's reference verdicts
