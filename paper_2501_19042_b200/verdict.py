"""Feasibility verdict and trajectory evaluation on the device (K2).

``feasible_results`` is the numerator of the headline metric (feasible
samples/s): converged AND every original constraint within ``tol``
(``metrics.py:57-69`` -> ``assembly.py:437-487``).  The margins are
evaluated in FP64 on the sampled trajectory C W^T by ``sgsf_verdict``; the
sampled trajectory itself (positions, velocities, accelerations,
``basis.py:149-160``) comes from ``sgsf_trajectory``.

``check_original_constraints`` is the reference's full report (``assembly.py:437-487``): counts, worst
margins and the worst-first violation lists, with the margins of ``problem.py:113-137`` evaluated on the
device in the reference's operation order (FP64, no contraction) and ordered by a stable device sort.
"""
from __future__ import annotations

from collections import OrderedDict
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
    """Original-constraint check of a trajectory (``assembly.py:410-433``): counts, worst margins and the
    worst-first lists (i, j, sample, margin) / (robot, sample, margin)."""

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


_CACHE_SIZE = 8   # operators (and their device constants) kept per cache: least recently used evicted
_OPS: OrderedDict = OrderedDict()


def _lru_get(cache: OrderedDict, key, make):
    hit = cache.get(key)
    if hit is None:
        hit = cache[key] = make()
        while len(cache) > _CACHE_SIZE:
            cache.popitem(last=False)
    cache.move_to_end(key)
    return hit[0]


def _operator(problem, degree: int) -> Operator:
    def make():
        basis = build_basis(problem.duration, degree=degree, samples=problem.horizon_samples)
        return Operator(problem, basis, build_equality(problem, basis)), problem   # (problem kept: id() unique)
    return _lru_get(_OPS, (id(problem), degree), make)


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
    cd = _to_dev(c.reshape(1, -1))
    v = {k: t.cpu().numpy()[0] for k, t in verdict_batched(op, cd, None, tol).items()}
    pl, wl = (), ()
    if not v["ok"]:   # the worst-first lists, from the device trajectory
        pos, _, _ = _trajectories(op.basis, problem.n, cd, host=False)
        rep = _check_positions(pos[0], problem, tol, 100)
        pl, wl = rep.pair_violations, rep.workspace_violations
    return ViolationReport(bool(v["ok"]), tol, float(v["pair_margin_min"]) if problem.n > 1 else np.inf,
                           float(v["ws_margin_max"]), int(v["pair_viol"]), int(v["ws_viol"]), pl, wl)


def _check_positions(pos: torch.Tensor, problem, tol: float, max_listed: int) -> ViolationReport:
    """check_original_constraints on device positions (n, S, 3) FP64: the margins of problem.py:113-137 as
    separate IEEE operations in the reference's order, counts, worst margins and worst-first lists."""
    n = int(pos.shape[0])
    if n != problem.n:
        raise DimensionMismatch(f"trajectory has {n} robots, problem expects {problem.n}")
    ws_ = problem.workspace
    d = pos - torch.as_tensor(np.asarray(ws_.center, dtype=float), device=pos.device)
    aw2, bw2 = float(ws_.lateral) ** 2, float(ws_.vertical) ** 2
    ws_m = ((d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) / aw2 + (d[..., 2] * d[..., 2]) / bw2) - 1.0
    bad = torch.nonzero(ws_m > tol)                                   # row-major, like np.argwhere
    vals = ws_m[bad[:, 0], bad[:, 1]]
    order = torch.sort(-vals, stable=True).indices[:max_listed]
    ws_list = [(int(r), int(t), float(m)) for (r, t), m in zip(bad[order].tolist(), vals[order].tolist())]
    n_ws = int(bad.shape[0])
    pair_list, pair_min, n_pair = [], np.inf, 0
    if n > 1:
        ii, jj = np.triu_indices(n, k=1)
        it, jt = (torch.as_tensor(a, device=pos.device) for a in (ii, jj))
        dl = pos[it] - pos[jt]
        a2, b2 = float(problem.shape.lateral) ** 2, float(problem.shape.vertical) ** 2
        pm = ((dl[..., 0] * dl[..., 0] + dl[..., 1] * dl[..., 1]) / a2 + (dl[..., 2] * dl[..., 2]) / b2) - 1.0
        pair_min = float(pm.min())
        bad = torch.nonzero(pm < -tol)
        vals = pm[bad[:, 0], bad[:, 1]]
        order = torch.sort(vals, stable=True).indices[:max_listed]
        pair_list = [(int(ii[p]), int(jj[p]), int(t), float(m))
                     for (p, t), m in zip(bad[order].tolist(), vals[order].tolist())]
        n_pair = int(bad.shape[0])
    return ViolationReport(n_pair == 0 and n_ws == 0, tol, pair_min if n > 1 else np.inf, float(ws_m.max()),
                           n_pair, n_ws, tuple(pair_list), tuple(ws_list))


def check_original_constraints(traj: Trajectory, problem, tol: float = 1e-3, max_listed: int = 100) -> ViolationReport:
    """The reference's original-constraint check of a sampled trajectory (assembly.py:437-487), on the device."""
    pos = np.asarray(traj.positions, dtype=float)
    if pos.ndim != 3 or pos.shape[0] != problem.n:
        raise DimensionMismatch(f"trajectory has {pos.shape[0] if pos.ndim else 0} robots, problem expects {problem.n}")
    return _check_positions(_to_dev(pos), problem, tol, max_listed)


def _trajectories(basis, n, cd: torch.Tensor, host: bool = True):
    """Sampled positions / velocities / accelerations (B, n, S, 3) of (B, dim) device coefficients: one launch
    (numpy when `host`, else the device tensors)."""
    from .solver import _to_host
    op = _trajectory_operator(basis, n)
    B, S = int(cd.shape[0]), basis.samples
    pos, vel, acc = (torch.empty((B, n, S, 3), dtype=torch.float64, device=cd.device) for _ in range(3))
    native.check(native.load().sgsf_trajectory(op.handle(1.0, cd.device), B, cd.data_ptr(), pos.data_ptr(),
                                               vel.data_ptr(), acc.data_ptr(), _stream()), "sgsf_trajectory")
    if not host:
        return pos, vel, acc
    h = _to_host({"p": pos, "v": vel, "a": acc})
    return h["p"], h["v"], h["a"]


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


_TRAJ: OrderedDict = OrderedDict()


def _trajectory_operator(basis, n) -> Operator:
    def make():
        prob = _BasisOnlyProblem(n, basis)
        return Operator(prob, basis, build_equality(prob, basis)), basis
    return _lru_get(_TRAJ, (id(basis), n), make)


def feasible_results(results, problem, tol: float = 1e-3) -> list:
    """(index, trajectory) of results that converged and pass the original constraints."""
    keep = [(i, r) for i, r in enumerate(results) if r.converged and r.coeffs is not None]
    if not keep:
        return []
    out = []
    by_degree: dict = {}   # (the reference takes each result's degree from its own coefficient count)
    for i, r in keep:
        by_degree.setdefault(r.coeffs.size // (3 * problem.n) - 1, []).append((i, r))
    for degree, group in by_degree.items():
        op = _operator(problem, degree)
        cd = _to_dev(np.stack([r.coeffs for _, r in group]))
        ok = verdict_batched(op, cd, None, tol)["ok"].cpu().numpy().astype(bool)
        if not ok.any():
            continue
        good = cd[torch.from_numpy(ok).to(cd.device)].contiguous()
        pos, vel, acc = _trajectories(op.basis, problem.n, good)
        k = 0
        for (i, _), g in zip(group, ok):
            if g:
                out.append((i, Trajectory(pos[k], vel[k], acc[k], op.basis.time_grid)))
                k += 1
    return sorted(out, key=lambda t: t[0])


def feasible_fraction(results, problem, tol: float = 1e-3):
    results = list(results)
    if not results:
        return None
    return len(feasible_results(results, problem, tol=tol)) / len(results)
