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


def test_cpu_stream_counts_until_min_samples():
    """The CPU baseline's pool (bench.CpuStream): a slice keeps counting past its time budget until `min_samples`
    proposals have completed (the 64-robot legs wait for a full wave), and reports the sample-iterations it saw."""
    sys.path.insert(0, str(REPO))
    import bench
    from paper_2501_19042_b200 import load_problem, sample_proposals
    from paper_2501_19042_b200.basis import build_basis
    from paper_2501_19042_b200.scenarios import random_swarm_doc
    doc = random_swarm_doc(2, 20, 1)
    prob = load_problem(doc)
    basis = build_basis(prob.duration, degree=10, samples=prob.horizon_samples)
    props = sample_proposals(prob, basis, 4, seed=0, spread=0.6).proposals
    stream = bench.CpuStream(doc, props, max_iters=30, cores=2)
    try:
        r = stream.take(0.0, min_samples=5)
    finally:
        stream.close()
    assert r["samples"] >= 5 and r["sample_iterations"] >= r["samples"] and r["wall_s"] > 0
