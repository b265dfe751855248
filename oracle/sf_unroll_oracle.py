"""CPU oracle for the differentiable safety filter (unrolled fixed-point steps and their gradient).

TEST INFRASTRUCTURE ONLY, like ``sf_oracle``: only ``tests/`` may import it; the product path
(``paper_2501_19042_b200.unrolled`` over ``sgsf_unroll`` / ``sgsf_unroll_backward``) never does.

The paper trains its initialisation network through K unrolled SF fixed-point steps
(PAPER.md "Learned Initialization for SF", eq. NN_loss).  The reference package has no autodiff, so the
oracle is torch FP64 autograd through a restatement of the reference step, built from the same pieces
as ``sf_oracle.solve`` (the loop body ``solver.py:314-328``):

* targets from the reference trig formula (``kernels/reference.py:13-48``: atan2 / hypot / sin / cos,
  clip of the radial), so autograd differentiates the reference's own expression, not the
  kernel's trig-free form;
* lambda' = lambda - rho F^T (F xi - E) (``solver.py:317-321``), eta = rho F^T E + lambda' + xi_bar
  (``solver.py:323-327``, workspace targets plus the centre);
* the xi-step as a dense solve of the 17n saddle system (``assembly.py:164-219``) with
  ``torch.linalg.solve`` (no refinement loop: its correction is below 1e-13 here).

Pinning: the forward iterates equal ``sf_oracle.solve`` (pinned to the reference's golden vectors) to
1e-11, and the gradient equals central finite differences of that forward
(``tests/test_unroll_oracle.py``).
"""
from __future__ import annotations

import numpy as np
import torch

from . import sf_oracle


class TorchProblem:
    """Torch FP64 constants of an ``sf_oracle.OracleProblem``."""

    def __init__(self, prob: sf_oracle.OracleProblem, rho: float = 1.0):
        self.prob = prob
        self.rho = float(rho)
        f = lambda a: torch.as_tensor(np.asarray(a, dtype=float), dtype=torch.float64)
        self.W = f(prob.W)
        self.inc = f(prob.incidence)
        self.pi = torch.as_tensor(prob.pair_i, dtype=torch.long)
        self.pj = torch.as_tensor(prob.pair_j, dtype=torch.long)
        self.ctr = f(prob.center).reshape(3, 1, 1)
        self.K = f(sf_oracle.kkt_matrix(prob, rho))
        self.rhs = f(prob.rhs)          # (3, n, 6)
        self.B = f(prob.endpoint)       # (6, m1)

    @property
    def shape(self):
        return (3, self.prob.n, self.prob.m1)


def spherical_targets(dx, dy, dz, lat, vert, lo, hi):
    """Reference trig formula (kernels/reference.py:13-48) in torch; returns the target (tx, ty, tz)."""
    az = torch.atan2(dy, dx)
    planar = torch.hypot(dx, dy)
    pol = torch.atan2(planar / lat, dz / vert)
    sp, cp = torch.sin(pol), torch.cos(pol)
    rad = torch.clamp((lat * sp * planar + vert * cp * dz) / ((lat * sp) ** 2 + (vert * cp) ** 2), min=lo, max=hi)
    lr = lat * rad * sp
    return lr * torch.cos(az), lr * torch.sin(az), vert * rad * cp


def transpose_apply(tp: TorchProblem, v_pair, v_ws):
    """F^T on per-block values (assembly.py:296-303)."""
    return (torch.einsum("pn,apt->ant", tp.inc, v_pair) + v_ws) @ tp.W


def step(tp: TorchProblem, C, lam, xb):
    """One fixed-point step (xi, lambda) -> (xi', lambda'), each (3, n, m1)."""
    p = tp.prob
    pos = C @ tp.W.T
    d = pos[:, tp.pi, :] - pos[:, tp.pj, :]
    rel = pos - tp.ctr
    pt = torch.stack(spherical_targets(d[0], d[1], d[2], p.lat, p.vert, 1.0, None))
    wt = torch.stack(spherical_targets(rel[0], rel[1], rel[2], p.ws_lat, p.ws_vert, 0.0, 1.0))
    lam_n = lam - tp.rho * transpose_apply(tp, d - pt, rel - wt)
    eta = tp.rho * transpose_apply(tp, pt, wt + tp.ctr) + lam_n + xb
    nc = p.n * p.m1
    rhs = torch.cat([eta.reshape(3, nc).T, tp.rhs.reshape(3, -1).T], dim=0)
    sol = torch.linalg.solve(tp.K, rhs)
    return sol[:nc].T.reshape(tp.shape), lam_n


def boundary_projection(tp: TorchProblem, xb):
    """xi - B^T (B B^T)^-1 (B xi - b) per robot and axis (projection.py:11-25)."""
    res = xb @ tp.B.T - tp.rhs
    y = torch.linalg.solve(tp.B @ tp.B.T, res.reshape(-1, 6).T)
    return xb - (y.T @ tp.B).reshape(xb.shape)


def unroll(tp: TorchProblem, xi_bar, xi0, lam0, iters: int):
    """Iterates (xs, ls), each (iters + 1, dim), from flat (dim,) tensors."""
    xb = xi_bar.reshape(tp.shape)
    C = xi0.reshape(tp.shape)
    lam = lam0.reshape(tp.shape)
    xs, ls = [C.reshape(-1)], [lam.reshape(-1)]
    for _ in range(iters):
        C, lam = step(tp, C, lam, xb)
        xs.append(C.reshape(-1))
        ls.append(lam.reshape(-1))
    return torch.stack(xs), torch.stack(ls)


def fixed_point_loss(xs, ls, xi_bar):
    """PAPER.md eq. NN_loss for one sample: sum_k ||z_{k+1} - z_k||^2 + ||xi_K - xi_bar||^2."""
    dz = torch.cat([xs[1:] - xs[:-1], ls[1:] - ls[:-1]], dim=1)
    return (dz * dz).sum() + ((xs[-1] - xi_bar) ** 2).sum()


def gradients(tp: TorchProblem, xi_bar, xi0, lam0, iters: int, gx, gl):
    """d/d(xi_bar, xi0, lam0) of sum(gx * xs) + sum(gl * ls) (numpy in and out)."""
    t = lambda a: torch.tensor(np.asarray(a, dtype=float), dtype=torch.float64, requires_grad=True)
    xb, x0, l0 = t(xi_bar), t(xi0), t(lam0)
    xs, ls = unroll(tp, xb, x0, l0, iters)
    loss = (xs * torch.as_tensor(gx)).sum() + (ls * torch.as_tensor(gl)).sum()
    loss.backward()
    return xb.grad.numpy(), x0.grad.numpy(), l0.grad.numpy(), xs.detach().numpy(), ls.detach().numpy()
