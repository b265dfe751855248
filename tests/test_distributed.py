"""Multi-process (world_size 2, gloo, CPU) tests of the shard / gather logic.

The solve itself needs a GPU; here each rank fabricates the outputs its shard
would produce (row-identifying values), and the test checks that the gather
reassembles the full batch in order on every rank.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2501_19042_b200.distributed import gather_outputs, shard_range


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, batch, dim, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_range(batch, world, rank)
        rows = torch.arange(lo, hi, dtype=torch.float64)
        out = {
            "coeffs": rows[:, None] * 10.0 + torch.arange(dim, dtype=torch.float64)[None, :],
            "iterations": (rows * 3).to(torch.int32),
            "converged": (rows.to(torch.int64) % 2).to(torch.uint8),
            "residual_inf": rows[:, None].repeat(1, 5),
        }
        g = gather_outputs(out, batch)
        full = torch.arange(batch, dtype=torch.float64)
        ok = (torch.equal(g["coeffs"], full[:, None] * 10.0 + torch.arange(dim, dtype=torch.float64)[None, :])
              and torch.equal(g["iterations"], (full * 3).to(torch.int32))
              and torch.equal(g["converged"], (full.to(torch.int64) % 2).to(torch.uint8))
              and g["residual_inf"].shape == (batch, 5))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch", [10, 7, 1])
def test_gather_reassembles_batch_world2(batch):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, batch, 4, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = dict(q.get(timeout=5) for _ in range(2))
    assert results == {0: True, 1: True}


def test_shard_range_partitions():
    for batch in (0, 1, 7, 1000):
        for world in (1, 2, 3, 8):
            spans = [shard_range(batch, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
