"""bench.py's multi-GPU plumbing on CPU: `--gpus N` outside torchrun relaunches itself as N ranks
(torch.distributed.run, 127.0.0.1), each rank takes its contiguous shard of the one global batch, the
per-sample outputs are all-gathered, the time is the max over ranks and rank 0 alone prints one line.
The solve is stubbed (`--stub`, gloo), so this runs without a GPU."""
import json
import subprocess
import sys

import pytest

from .conftest import REPO


@pytest.mark.parametrize("config,gpus,per_gpu", [(2, 2, 1000), (3, 2, 2048)])
def test_gpus_flag_launches_ranks(config, gpus, per_gpu):
    r = subprocess.run([sys.executable, str(REPO / "bench.py"), "--gpus", str(gpus), "--stub", "--config", str(config),
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=REPO)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout   # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == gpus and d["stub"]
    assert d["config"]["batch_per_gpu"] == per_gpu
    # weak scaling for config 2 (1000 per GPU), strong for config 3 (4096 over the ranks)
    assert d["config"]["batch"] == (1000 * gpus if config == 2 else 4096)
    assert d["scaling"] == ("weak" if config == 2 else "strong")
