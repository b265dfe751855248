"""The differentiable safety filter: K unrolled fixed-point steps and their gradient, on the GPU.

The paper trains its initialisation network through an unrolled chain of K SF fixed-point steps
z_{k+1} = f_FP(z_k), z = (xi, lambda) (PAPER.md "Learned Initialization for SF", eq. NN_loss;
BASELINE config 5).  The reference package has no autodiff; the step is its solve-loop body
(``solver.py:314-328``).  Both directions run in ``libsgsf.so`` in FP64:

* ``sgsf_unroll`` writes every iterate (no early stop);
* ``sgsf_unroll_backward`` is the exact vector-Jacobian product of the chain.

Both are in ``csrc/kernels_unroll.cu``, one CTA per sample.  :func:`unrolled_solve` wraps them as a
``torch.autograd.Function``, so any torch loss on the iterates (e.g. :func:`fixed_point_loss`)
backpropagates into the proposal and the initialisation.
"""
from __future__ import annotations

from typing import NamedTuple

import torch

from . import native
from .errors import DimensionMismatch


class UnrolledIterates(NamedTuple):
    coeffs: torch.Tensor        # (B, K + 1, dim): xi_0 .. xi_K
    multipliers: torch.Tensor   # (B, K + 1, dim): lambda_0 .. lambda_K


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


class _Unrolled(torch.autograd.Function):
    @staticmethod
    def forward(ctx, xi_bar, xi0, lam0, handle, iters):
        B, dim = xi_bar.shape
        xs = torch.empty((B, iters + 1, dim), dtype=torch.float64, device=xi_bar.device)
        ls = torch.empty_like(xs)
        native.check(native.load().sgsf_unroll(handle, B, iters, xi_bar.data_ptr(), xi0.data_ptr(),
                                               lam0.data_ptr(), xs.data_ptr(), ls.data_ptr(), _stream()),
                     "sgsf_unroll")
        ctx.save_for_backward(xs)
        ctx.handle = handle
        ctx.iters = iters
        return xs, ls

    @staticmethod
    @torch.autograd.function.once_differentiable
    def backward(ctx, gxs, gls):
        (xs,) = ctx.saved_tensors
        B, _, dim = xs.shape
        gx = gxs.contiguous() if gxs is not None else None
        gl = gls.contiguous() if gls is not None else None
        g_xb = torch.empty((B, dim), dtype=torch.float64, device=xs.device)
        g_x0 = torch.empty_like(g_xb)
        g_l0 = torch.empty_like(g_xb)
        native.check(native.load().sgsf_unroll_backward(ctx.handle, B, ctx.iters, xs.data_ptr(), native.ptr(gx),
                                                        native.ptr(gl), g_xb.data_ptr(), g_x0.data_ptr(),
                                                        g_l0.data_ptr(), _stream()),
                     "sgsf_unroll_backward")
        return g_xb, g_x0, g_l0, None, None


def device_constants_of(sf, device) -> dict:
    """Per-(filter, device) cache of the small constants the torch-side layers need (boundary rows,
    projector, endpoint rhs, straight-line coefficients, start/goal context), uploaded once so the
    decoder -> QP layer -> SF pipeline makes no host transfers per call."""
    cache = sf.__dict__.setdefault("_device_consts", {})
    key = (str(torch.device(device)), float(sf.config.rho))
    if key not in cache:
        from .initnet import context_features
        from .proposals import straight_line_coeffs
        k = sf.operator.constants(sf.config.rho)
        f64 = dict(dtype=torch.float64, device=device)
        cache[key] = {
            "B": torch.as_tensor(k.B, **f64), "PBt": torch.as_tensor(k.PBt, **f64),
            "rhs": torch.as_tensor(k.rhs, **f64), "n": k.n, "m1": k.m1,
            "base": torch.as_tensor(straight_line_coeffs(sf.problem, sf.basis), **f64),
            "context": torch.as_tensor(context_features(sf.problem), **f64),
        }
        cache[key]["context32"] = cache[key]["context"].to(torch.float32)   # (the decoders' input dtype)
    return cache[key]


def boundary_projection(sf, xi_bar: torch.Tensor) -> torch.Tensor:
    """The default start xi_0 = xi_bar - B^T (B B^T)^-1 (B xi_bar - b) per robot and axis
    (``projection.py:11-25``) as torch ops, so gradients reach the proposal through it."""
    k = device_constants_of(sf, xi_bar.device)
    Bm, PBt, rhs = k["B"], k["PBt"], k["rhs"]   # (6, m1), (m1, 6), (3, n, 6)
    C = xi_bar.reshape(xi_bar.shape[0], 3, k["n"], k["m1"])
    res = C @ Bm.T - rhs
    return (C - res @ PBt.T).reshape(xi_bar.shape)


def unrolled_solve(sf, xi_bar: torch.Tensor, xi0: torch.Tensor | None = None, lam0: torch.Tensor | None = None,
                   iters: int = 10, rho: float | None = None) -> UnrolledIterates:
    """``iters`` SF fixed-point steps of a (B, dim) float64 CUDA batch, differentiable with respect to
    ``xi_bar``, ``xi0`` and ``lam0``.  The default start is the boundary projection of the proposal
    with zero multipliers (``solver.py:264-284``), the same as :meth:`SafetyFilter.solve_batched`."""
    dim = sf.coeff_dim
    if xi_bar.dim() != 2 or xi_bar.shape[1] != dim:
        raise DimensionMismatch(f"proposals must be (B, {dim}), got {tuple(xi_bar.shape)}")
    if not xi_bar.is_cuda or xi_bar.dtype != torch.float64:
        raise DimensionMismatch("proposals must be a float64 CUDA tensor")
    if iters < 0:
        raise ValueError(f"iters must be >= 0, got {iters}")
    for name, t in (("xi0", xi0), ("lam0", lam0)):
        if t is not None and (t.shape != xi_bar.shape or t.dtype != torch.float64 or t.device != xi_bar.device):
            raise DimensionMismatch(f"{name} must be a float64 tensor shaped like the proposals")
    if xi0 is None:
        xi0 = boundary_projection(sf, xi_bar)
    if lam0 is None:
        lam0 = torch.zeros_like(xi_bar)
    rho = sf.config.rho if rho is None else float(rho)
    handle = sf.operator.handle(rho, xi_bar.device)
    xs, ls = _Unrolled.apply(xi_bar.contiguous(), xi0.contiguous(), lam0.contiguous(), handle, int(iters))
    return UnrolledIterates(xs, ls)


def fixed_point_loss(it: UnrolledIterates, xi_bar: torch.Tensor, reduction: str = "mean") -> torch.Tensor:
    """PAPER.md eq. NN_loss per sample: the fixed-point residuals along the chain,
    sum_k ||z_{k+1} - z_k||^2 (the paper's ||z_{k+1} - f_FP(z_k)||^2 read as the learned-warm-start
    fixed-point residual, z_{k+1} = f_FP(z_k)), plus the displacement ||xi_K - xi_bar||^2."""
    xs, ls = it.coeffs, it.multipliers
    dz = torch.cat([xs[:, 1:] - xs[:, :-1], ls[:, 1:] - ls[:, :-1]], dim=2)
    per = (dz * dz).sum(dim=(1, 2)) + ((xs[:, -1] - xi_bar) ** 2).sum(dim=1)
    if reduction == "mean":
        return per.mean()
    if reduction == "sum":
        return per.sum()
    if reduction == "none":
        return per
    raise ValueError(f"reduction must be 'mean', 'sum' or 'none', got {reduction!r}")
