"""Feasibility verdict and trajectory evaluation on the device (K2).

``feasible_results`` is the numerator of the headline metric (feasible
samples/s): converged AND every original constraint within ``tol``
(``metrics.py:57-69`` -> ``assembly.py:437-487``).  The margins are
evaluated in FP64 on the sampled trajectory C W^T by ``sgsf_verdict``; the
sampled trajectory itself (positions, velocities, accelerations,
``basis.py:149-160``) comes from ``sgsf_trajectory``.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import native
from .basis import Trajectory, build_basis
from .errors import DimensionMismatch
from .precompute import build_equality
from .solver import Operator, _stream, _to_dev


@dataclass(frozen=True)
class ViolationReport:
    """Counts and worst margins (the reference also lists the worst violations;
    those lists are left empty here)."""

    ok: bool
    tol: float
    pair_margin_min: float
    workspace_margin_max: float
    pair_violation_count: int
    workspace_violation_count: int
    pair_violations: tuple = ()
    workspace_violations: tuple = ()

    def to_jsonable(self) -> dict:
        return {"ok": self.ok, "tol": self.tol, "pair_margin_min": self.pair_margin_min,
                "workspace_margin_max": self.workspace_margin_max,
                "pair_violation_count": self.pair_violation_count,
                "workspace_violation_count": self.workspace_violation_count,
                "pair_violations": [list(v) for v in self.pair_violations],
                "workspace_violations": [list(v) for v in self.workspace_violations]}


_OPS: dict = {}


def _operator(problem, degree: int) -> Operator:
    key = (id(problem), degree)
    op = _OPS.get(key)
    if op is None:
        basis = build_basis(problem.duration, degree=degree, samples=problem.horizon_samples)
        op = Operator(problem, basis, build_equality(problem, basis))
        _OPS[key] = (op, problem)   # keep the problem alive so id() stays unique
        return op
    return op[0]


def verdict_batched(operator: Operator, coeffs: torch.Tensor, converged: torch.Tensor | None = None,
                    tol: float = 1e-3) -> dict:
    """Device verdict for (B, dim) float64 CUDA coefficients; returns device tensors."""
    B = int(coeffs.shape[0])
    dev = coeffs.device
    out = {"ok": torch.empty(B, dtype=torch.uint8, device=dev),
           "feasible": torch.empty(B, dtype=torch.uint8, device=dev),
           "pair_margin_min": torch.empty(B, dtype=torch.float64, device=dev),
           "ws_margin_max": torch.empty(B, dtype=torch.float64, device=dev),
           "pair_viol": torch.empty(B, dtype=torch.int32, device=dev),
           "ws_viol": torch.empty(B, dtype=torch.int32, device=dev)}
    if B:
        v = native.Verdict(*(out[k].data_ptr() for k in ("ok", "feasible", "pair_margin_min", "ws_margin_max",
                                                          "pair_viol", "ws_viol")))
        native.check(native.load().sgsf_verdict(operator.handle(1.0, dev), B, coeffs.contiguous().data_ptr(),
                                                native.ptr(converged), float(tol), native.C.byref(v), _stream()),
                     "sgsf_verdict")
    return out


def check_coefficients(coeffs, problem, degree: int = 10, tol: float = 1e-3) -> ViolationReport:
    """Original-constraint check of one flat coefficient vector."""
    op = _operator(problem, degree)
    c = np.asarray(coeffs, dtype=float).ravel()
    if c.size != op.coeff_dim:
        raise DimensionMismatch(f"coefficient vector has length {c.size}, expected {op.coeff_dim}")
    v = {k: t.cpu().numpy()[0] for k, t in verdict_batched(op, _to_dev(c.reshape(1, -1)), None, tol).items()}
    return ViolationReport(bool(v["ok"]), tol, float(v["pair_margin_min"]) if problem.n > 1 else np.inf,
                           float(v["ws_margin_max"]), int(v["pair_viol"]), int(v["ws_viol"]))


def coeffs_to_trajectory(coeffs, basis, n) -> Trajectory:
    """Sample a flat coefficient vector on the basis grid (device evaluation)."""
    from .precompute import build_equality  # noqa: F401  (kept for symmetry with the reference module)
    c = np.asarray(coeffs, dtype=float).ravel()
    dim = 3 * n * (basis.degree + 1)
    if c.size != dim:
        raise DimensionMismatch(f"coefficient vector has length {c.size}, expected {dim} "
                                f"(n={n}, degree={basis.degree})")
    op = _trajectory_operator(basis, n)
    cd = _to_dev(c.reshape(1, -1))
    S = basis.samples
    pos, vel, acc = (torch.empty((1, n, S, 3), dtype=torch.float64, device=cd.device) for _ in range(3))
    native.check(native.load().sgsf_trajectory(op.handle(1.0, cd.device), 1, cd.data_ptr(), pos.data_ptr(),
                                               vel.data_ptr(), acc.data_ptr(), _stream()), "sgsf_trajectory")
    return Trajectory(pos.cpu().numpy()[0], vel.cpu().numpy()[0], acc.cpu().numpy()[0], basis.time_grid)


class _BasisOnlyProblem:
    """Minimal problem for trajectory evaluation (no constraints needed)."""

    def __init__(self, n, basis):
        from .problem import EndpointState, RobotBoundary, RobotShape, Workspace
        self.n = n
        self.horizon_samples = basis.samples
        self.duration = basis.duration
        self.shape = RobotShape(1.0, 1.0)
        self.workspace = Workspace(np.zeros(3), 1.0, 1.0)
        z = EndpointState(np.zeros(3))
        self.boundary = tuple(RobotBoundary(z, z) for _ in range(n))


_TRAJ: dict = {}


def _trajectory_operator(basis, n) -> Operator:
    key = (id(basis), n)
    hit = _TRAJ.get(key)
    if hit is None:
        prob = _BasisOnlyProblem(n, basis)
        hit = (Operator(prob, basis, build_equality(prob, basis)), basis)
        _TRAJ[key] = hit
    return hit[0]


def feasible_results(results, problem, tol: float = 1e-3) -> list:
    """(index, trajectory) of results that converged and pass the original constraints."""
    keep = [(i, r) for i, r in enumerate(results) if r.converged and r.coeffs is not None]
    if not keep:
        return []
    degree = keep[0][1].coeffs.size // (3 * problem.n) - 1
    op = _operator(problem, degree)
    cd = _to_dev(np.stack([r.coeffs for _, r in keep]))
    ok = verdict_batched(op, cd, None, tol)["ok"].cpu().numpy()
    return [(i, coeffs_to_trajectory(r.coeffs, op.basis, problem.n)) for (i, r), good in zip(keep, ok) if good]


def feasible_fraction(results, problem, tol: float = 1e-3):
    results = list(results)
    if not results:
        return None
    return len(feasible_results(results, problem, tol=tol)) / len(results)
