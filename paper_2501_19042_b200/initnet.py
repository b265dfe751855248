"""Learned SF initialisation, trained through the differentiable SF (BASELINE config 5).

PAPER.md "Learned Initialization for SF" and "Initialization Network Details":
* A PointNet-like CNN with 18 input channels (start and goal position, velocity and acceleration of
  each robot) gives a context feature c. It uses shared 1x1 convolutions over the robots and a max
  pool, so it is permutation invariant.
* c is concatenated with the proposal xi_bar.
* A 4-layer MLP (linear, LeakyReLU, batch norm) predicts the initialisation (xi_0, lambda_0).
* Training minimises eq. NN_loss (:func:`unrolled.fixed_point_loss`) through K unrolled SF steps. The
  steps run as the CUDA forward / reverse kernels of :mod:`unrolled`, so the gradient reaches the
  network through the SF itself.

The network is plain PyTorch: it is the learnable part of the pipeline, not the hot path.  The
reference ships no network, so there is no parity target. :func:`init_sweep` measures what
the net buys: SF iterations to the residual tolerance from each initialisation strategy (the paper's
"Validating the Efficacy of SF Initialization Network" comparison).
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field, replace

import numpy as np
import torch
from torch import nn

from .unrolled import boundary_projection, fixed_point_loss, unrolled_solve

STRATEGIES = ("zero", "proposal", "projected", "initnet")


def context_features(problem) -> np.ndarray:
    """(18, n): per robot [start p, v, a, goal p, v, a] as the CNN's input channels."""
    cols = []
    for rb in problem.boundary:
        cols.append(np.concatenate([rb.start.position, rb.start.velocity, rb.start.acceleration,
                                    rb.goal.position, rb.goal.velocity, rb.goal.acceleration]))
    return np.stack(cols, axis=1).astype(np.float64)


class InitNet(nn.Module):
    """PointNet-style context encoder + 4-layer MLP -> (xi_0, lambda_0).

    The last layer starts at zero and the coefficient output is a correction to the proposal. An
    untrained net therefore starts the SF from the raw proposal with zero multipliers (the "proposal"
    strategy), and training moves it from there.
    """

    def __init__(self, n: int, dim: int, width: int = 128, hidden: int = 512, slope: float = 0.01):
        super().__init__()
        self.n, self.dim = n, dim
        act = lambda: nn.LeakyReLU(slope)
        self.point = nn.Sequential(
            nn.Conv1d(18, 64, 1), nn.BatchNorm1d(64), act(),
            nn.Conv1d(64, 128, 1), nn.BatchNorm1d(128), act(),
            nn.Conv1d(128, width, 1))
        self.mlp = nn.Sequential(
            nn.Linear(width + dim, hidden), nn.BatchNorm1d(hidden), act(),
            nn.Linear(hidden, hidden), nn.BatchNorm1d(hidden), act(),
            nn.Linear(hidden, hidden), nn.BatchNorm1d(hidden), act(),
            nn.Linear(hidden, 2 * dim))
        nn.init.zeros_(self.mlp[-1].weight)
        nn.init.zeros_(self.mlp[-1].bias)

    def forward(self, context: torch.Tensor, xi_bar: torch.Tensor):
        """context (B, 18, n), xi_bar (B, dim) -> (xi_0, lambda_0), float64 like xi_bar."""
        c = self.point(context.to(self.mlp[0].weight.dtype)).amax(dim=2)
        out = self.mlp(torch.cat([c, xi_bar.to(c.dtype)], dim=1)).to(xi_bar.dtype)
        return xi_bar + out[:, :self.dim], out[:, self.dim:]


class FoldedInitNet:
    """The eval-mode init net for ONE problem as four cuBLAS GEMMs: the context encoder's output is the same
    for every sample of a problem, so it becomes a constant bias of the first layer (W1 [c | x] = W1_x x +
    W1_c c), and each batch norm folds into its Linear.  ``__call__(xi_bar)`` returns what
    ``net(context, xi_bar)`` returns (eval mode) to FP32 rounding, without the per-call PointNet pass,
    concatenation and normalisation kernels."""

    def __init__(self, net: InitNet, context: torch.Tensor):
        net = net.eval()
        self.dim = net.dim
        lin = [m for m in net.mlp if isinstance(m, nn.Linear)]
        bns = [m for m in net.mlp if isinstance(m, nn.BatchNorm1d)]
        acts = [m for m in net.mlp if isinstance(m, nn.LeakyReLU)]
        self.slope = float(acts[0].negative_slope)
        with torch.no_grad(), torch.backends.cudnn.flags(enabled=True, allow_tf32=False):
            c = net.point(context[:1].to(lin[0].weight.dtype)).amax(dim=2)[0].double()   # (width,)
            width = c.shape[0]
            self.W, self.b = [], []
            for i, L_ in enumerate(lin):
                W, b = L_.weight.double(), L_.bias.double()
                if i == 0:   # the context half of the first layer is a constant: fold it into the bias
                    b = b + W[:, :width] @ c
                    W = W[:, width:]
                if i < len(bns):
                    bn = bns[i]
                    sc = bn.weight.double() / torch.sqrt(bn.running_var.double() + bn.eps)
                    W = W * sc[:, None]
                    b = (b - bn.running_mean.double()) * sc + bn.bias.double()
                self.W.append(W.t().contiguous().float())   # (in, out) for x @ W
                self.b.append(b.float().contiguous())

    @torch.no_grad()
    def __call__(self, xi_bar: torch.Tensor):
        h = xi_bar.to(torch.float32)
        for i, (W, b) in enumerate(zip(self.W, self.b)):
            h = torch.addmm(b, h, W)
            if i < len(self.W) - 1:
                h = torch.nn.functional.leaky_relu(h, self.slope)
        out = h.to(xi_bar.dtype)
        return xi_bar + out[:, :self.dim], out[:, self.dim:]


@dataclass
class TrainLog:
    losses: list = field(default_factory=list)
    seconds: float = 0.0
    sf_seconds: float = 0.0     # device time in the unrolled SF forward + backward (CUDA events)
    steps: int = 0


def train_init_net(sf, net: InitNet, proposals: torch.Tensor, iters: int = 10, steps: int = 200,
                   batch: int = 256, lr: float = 1e-3, seed: int = 0) -> TrainLog:
    """Self-supervised training on a (N, dim) float64 CUDA pool of proposals of one problem."""
    return train_init_net_multi([(sf, proposals)], net, iters=iters, steps=steps, batch=batch, per_step=1, lr=lr,
                                seed=seed)


def train_init_net_multi(scenarios, net: InitNet, iters: int = 10, steps: int = 200, batch: int = 256,
                         per_step: int = 4, lr: float = 1e-3, seed: int = 0) -> TrainLog:
    """Training over several problems of the same shape (n, degree, horizon): ``scenarios`` is a list of
    (SafetyFilter, (N, dim) proposal pool) pairs.  Every step mixes ``per_step`` scenarios (round-robin)
    in one network batch, so the batch-norm statistics see several contexts, as they will at evaluation;
    each scenario's slice then runs through its own unrolled SF.  The network learns a start/goal-
    context-specific initialisation (PAPER.md "Learned Initialization for SF")."""
    dev = scenarios[0][1].device
    net.to(dev).train()
    ctxs = [torch.as_tensor(context_features(sf.problem), device=dev) for sf, _ in scenarios]
    opt = torch.optim.Adam(net.parameters(), lr=lr)
    gen = torch.Generator(device="cpu").manual_seed(seed)
    log = TrainLog()
    t0 = time.perf_counter()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sub = max(1, batch // per_step)
    for k in range(steps):
        picks = [(k * per_step + u) % len(scenarios) for u in range(per_step)]
        xbs, cs = [], []
        for s_i in picks:
            pool = scenarios[s_i][1]
            idx = torch.randint(0, pool.shape[0], (min(sub, pool.shape[0]),), generator=gen).to(dev)
            xbs.append(pool[idx])
            cs.append(ctxs[s_i].expand(xbs[-1].shape[0], -1, -1))
        xi0, lam0 = net(torch.cat(cs), torch.cat(xbs))
        start.record()
        loss, o = 0.0, 0
        for s_i, xb in zip(picks, xbs):
            m = xb.shape[0]
            it = unrolled_solve(scenarios[s_i][0], xb, xi0[o:o + m], lam0[o:o + m], iters=iters)
            loss = loss + fixed_point_loss(it, xb, reduction="sum")
            o += m
        loss = loss / o
        opt.zero_grad(set_to_none=True)
        loss.backward()
        stop.record()
        opt.step()
        stop.synchronize()
        log.sf_seconds += start.elapsed_time(stop) / 1e3
        log.losses.append(float(loss.detach()))
        log.steps += 1
    log.seconds = time.perf_counter() - t0
    return log


def initial_states(sf, proposals: torch.Tensor, strategy: str, net: InitNet | None = None):
    """(xi_0, lambda_0) of one strategy: zero vectors, the raw proposal, its boundary projection (the
    reference default, solver.py:264-284), or the init net's prediction."""
    zeros = torch.zeros_like(proposals)
    if strategy == "zero":
        return zeros, zeros.clone()
    if strategy == "proposal":
        return proposals.clone(), zeros
    if strategy == "projected":
        return boundary_projection(sf, proposals), zeros
    if strategy == "initnet":
        if net is None:
            raise ValueError("strategy 'initnet' needs a network")
        if isinstance(net, FoldedInitNet):
            return net(proposals)
        net.eval()
        with torch.no_grad():
            from .unrolled import device_constants_of
            ctx = device_constants_of(sf, proposals.device)["context"]
            return net(ctx.expand(proposals.shape[0], -1, -1), proposals)
    raise ValueError(f"unknown strategy {strategy!r}; choose from {list(STRATEGIES)}")


def init_sweep(sf, proposals: torch.Tensor, net: InitNet | None = None, strategies=STRATEGIES,
               max_iters: int = 500, trace_iters: int = 100) -> dict:
    """Per strategy, on the device solver:
    * mean and median iterations to the residual tolerance;
    * converged and feasible fractions;
    * the mean inf-norm residual per iteration over the first ``trace_iters`` iterations, run with
      early stop off (PAPER.md Fig. res)."""
    out = {}
    for s in strategies:
        if s == "initnet" and net is None:
            continue
        xi0, lam0 = initial_states(sf, proposals, s, net)
        cfg = replace(sf.config, max_iters=max_iters, svars=False)
        res = sf.solve_batched(proposals, xi0=xi0, lam0=lam0, config=cfg)
        its = res.iterations.double()
        trace = sf.solve_batched(proposals, xi0=xi0, lam0=lam0, verdict=False,
                                 config=replace(cfg, max_iters=trace_iters, early_stop=False))
        out[s] = {
            "mean_iterations": float(its.mean()),
            "median_iterations": float(its.median()),
            "converged": float(res.converged.double().mean()),
            "feasible": float(res.feasible.double().mean()) if res.feasible is not None else None,
            "residual_trace": trace.residual_inf.mean(dim=0).cpu().numpy().tolist(),
        }
    return out
