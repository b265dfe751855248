"""Multi-GPU batch filtering: contiguous sample shards, outputs gathered over NCCL.

Samples are independent, so the solve itself needs no communication (SURVEY
8e): rank r filters rows [lo_r, hi_r) of the batch on its own GPU with one
persistent-kernel launch, then the per-sample outputs (projected coefficients,
multipliers, residual histories, iterations, verdicts) are all-gathered so
every rank -- or the caller on rank 0 -- holds the full batch.  Every rank
builds identical device constants from the same FP64 host precompute, so
nothing is broadcast.  One process per GPU (torchrun); the process group is
NCCL for CUDA tensors and gloo for the CPU tests of the shard/gather logic.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

GATHERED_FIELDS = ("coeffs", "multipliers", "residual_inf", "residual_l2", "iterations", "converged", "feasible",
                   "displacement", "status")


def shard_range(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of `batch` rows for `rank` of `world`; sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(batch, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_rows(t: torch.Tensor, batch: int, group=None) -> torch.Tensor:
    """All-gather the row shards of `t` (this rank's [lo, hi) rows) into the full (batch, ...) tensor."""
    world = dist.get_world_size(group)
    cap = -(-batch // world)                     # ceil: every rank sends the same padded size
    pad = torch.zeros((cap,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    if dist.get_backend(group) == "nccl":
        full = torch.empty((world * cap,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(full, pad.contiguous(), group=group)
        parts = list(full.split(cap))
    else:
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
    rows = [parts[r][: hi - lo] for r, (lo, hi) in ((r, shard_range(batch, world, r)) for r in range(world))]
    return torch.cat(rows, dim=0)


def gather_outputs(out, batch: int, group=None) -> dict:
    """Gather the per-sample outputs of a DeviceBatch-like object (attributes or dict)."""
    get = (lambda k: out[k]) if isinstance(out, dict) else (lambda k: getattr(out, k))
    res = {}
    for k in GATHERED_FIELDS:
        try:
            t = get(k)
        except (KeyError, AttributeError):
            continue
        if t is not None:
            res[k] = gather_rows(t, batch, group)
    return res


def gather_outputs_async(out, batch: int, group=None):
    """gather_outputs without blocking the calling stream: NCCL all-gathers issued with async_op=True (their
    kernels run on the process group's stream; the caller's stream does not wait for them, so the next batch
    on it is not queued behind a collective that needs an SM).  Returns finish() -> the gathered dict, which
    makes the current stream wait for the collectives.  Equal shards only (batch divisible by the world size:
    no padding kernel); otherwise it gathers synchronously."""
    world = dist.get_world_size(group)
    if dist.get_backend(group) != "nccl" or batch % world:
        res = gather_outputs(out, batch, group)
        return lambda: res
    get = (lambda k: out[k]) if isinstance(out, dict) else (lambda k: getattr(out, k))
    pend = []
    for k in GATHERED_FIELDS:
        try:
            t = get(k)
        except (KeyError, AttributeError):
            continue
        if t is None:
            continue
        t = t.contiguous()
        full = torch.empty((batch,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pend.append((k, full, dist.all_gather_into_tensor(full, t, group=group, async_op=True)))

    def finish() -> dict:
        for _, _, work in pend:
            work.wait()
        return {k: full for k, full, _ in pend}
    return finish


def sharded_solve(sf, xi_bar: torch.Tensor, config=None, group=None, **kw) -> dict:
    """Filter a full (B, dim) batch across the ranks of `group`; every rank returns the full outputs.

    `xi_bar` may live on the host or any device; each rank copies only its shard
    to its own GPU.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    batch = int(xi_bar.shape[0])
    lo, hi = shard_range(batch, world, rank)
    dev = torch.device("cuda", torch.cuda.current_device())
    shard = xi_bar[lo:hi].to(dev, dtype=torch.float64, non_blocking=True).contiguous()
    out = sf.solve_batched(shard, config=config, **kw)
    return gather_outputs(out, batch, group)
