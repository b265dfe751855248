"""CPU oracle for the Swarm-Gen safety filter (SF) hot path.

TEST INFRASTRUCTURE ONLY.  This module is the checker, never the product:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import it.  The
product path (``paper_2501_19042_b200``) never imports, calls or links it.

It is a plain numpy/scipy FP64 restatement of the reference algorithm
(``/root/reference/pkg/src/swarmfilter``), written so that it keeps the
reference's arithmetic: atan2/hypot/sin/cos spherical projection, the dense
17n x 17n saddle-point LU factorisation with the same refinement loop, the
same per-iteration order of operations.  Every function cites the reference
``file:line`` it follows.

Parity is pinned: ``tests/test_oracle.py`` checks this module against the
golden vectors in ``tests/golden/`` that ``tests/golden/make_golden.py``
produced by importing and running the real reference in the build container.

Problems are passed as plain JSON-style dicts with the reference schema
(``problem.py:217-283``: n, H, T, a, b, workspace{center,a_w,b_w},
boundary[{start{p,v,a}, goal{p,v,a}}]) so the oracle stays independent of the
package under test.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from math import comb

import numpy as np
import scipy.linalg


# --------------------------------------------------------------------------- basis
def bernstein_basis(degree: int, samples: int, duration: float):
    """Value / velocity / acceleration sampling matrices, each (samples, degree+1).

    Follows ``basis.py:25-69`` (binomial * s^k * (1-s)^(m-k) on a linspace
    grid; derivatives from the degree-lowered basis times m/T and m(m-1)/T^2).
    """
    s = np.linspace(0.0, duration, samples) / duration

    def raw(m):
        k = np.arange(m + 1)
        coef = np.array([comb(m, int(j)) for j in k], dtype=float)
        return coef[None, :] * s[:, None] ** k[None, :] * (1.0 - s[:, None]) ** (m - k)[None, :]

    W = raw(degree)
    lo1 = raw(degree - 1)
    Wd = np.zeros_like(W)
    Wd[:, :-1] -= lo1
    Wd[:, 1:] += lo1
    Wd *= degree / duration
    Wdd = np.zeros_like(W)
    if degree >= 2:
        lo2 = raw(degree - 2)
        Wdd[:, :-2] += lo2
        Wdd[:, 1:-1] -= 2.0 * lo2
        Wdd[:, 2:] += lo2
        Wdd *= degree * (degree - 1) / duration ** 2
    return W, Wd, Wdd


# --------------------------------------------------------------------------- problem
@dataclass
class OracleProblem:
    """Everything the SF loop needs for one (problem, degree) pair."""

    n: int
    samples: int
    degree: int
    lat: float
    vert: float
    ws_lat: float
    ws_vert: float
    center: np.ndarray
    W: np.ndarray
    Wd: np.ndarray
    Wdd: np.ndarray
    endpoint: np.ndarray          # (6, m1): rows p0 v0 a0 pT vT aT   (assembly.py:42-53)
    rhs: np.ndarray               # (3, n, 6)                          (assembly.py:120-130)
    pair_i: np.ndarray
    pair_j: np.ndarray
    incidence: np.ndarray         # (P, n)                             (assembly.py:235-241)
    _kkt: dict = field(default_factory=dict, repr=False)

    @property
    def m1(self) -> int:
        return self.degree + 1

    @property
    def dim(self) -> int:
        return 3 * self.n * self.m1


def make_problem(doc: dict, degree: int = 10) -> OracleProblem:
    """Build an OracleProblem from a reference-schema problem dict (problem.py:217-283)."""
    n = int(doc["n"])
    samples = int(doc["H"]) + 1
    duration = float(doc["T"])
    W, Wd, Wdd = bernstein_basis(degree, samples, duration)
    endpoint = np.vstack([W[0], Wd[0], Wdd[0], W[-1], Wd[-1], Wdd[-1]])
    rhs = np.zeros((3, n, 6))
    for i, rb in enumerate(doc["boundary"]):
        st, gl = rb["start"], rb["goal"]
        for ax in range(3):
            rhs[ax, i] = (
                st["p"][ax], st.get("v", [0.0] * 3)[ax], st.get("a", [0.0] * 3)[ax],
                gl["p"][ax], gl.get("v", [0.0] * 3)[ax], gl.get("a", [0.0] * 3)[ax],
            )
    pi, pj = np.triu_indices(n, k=1)
    inc = np.zeros((pi.size, n))
    inc[np.arange(pi.size), pi] = 1.0
    inc[np.arange(pi.size), pj] = -1.0
    ws = doc["workspace"]
    return OracleProblem(
        n=n, samples=samples, degree=degree,
        lat=float(doc["a"]), vert=float(doc["b"]),
        ws_lat=float(ws["a_w"]), ws_vert=float(ws["b_w"]),
        center=np.asarray(ws["center"], dtype=float),
        W=W, Wd=Wd, Wdd=Wdd, endpoint=endpoint, rhs=rhs,
        pair_i=pi, pair_j=pj, incidence=inc,
    )


# --------------------------------------------------------------------------- pieces
def spherical_project(dx, dy, dz, lat, vert, lo, hi):
    """Closed-form spherical block update, reference trig formula.

    Follows ``kernels/reference.py:13-48`` (== ``_speedups.pyx:18-73``):
    az = atan2(dy, dx); pol = atan2(hypot(dx,dy)/lat, dz/vert) with the
    all-zero input mapped to pi/2; rad = clip(num/den, lo, hi); target from
    (az, pol, rad).  Returns (az, pol, rad, tx, ty, tz).
    """
    dx = np.asarray(dx, dtype=float)
    dy = np.asarray(dy, dtype=float)
    dz = np.asarray(dz, dtype=float)
    az = np.arctan2(dy, dx)
    planar = np.hypot(dx, dy)
    pol = np.arctan2(planar / lat, dz / vert)
    pol = np.where((planar == 0.0) & (dz == 0.0), 0.5 * np.pi, pol)
    sp, cp = np.sin(pol), np.cos(pol)
    rad = np.clip((lat * sp * planar + vert * cp * dz)
                  / ((lat * sp) ** 2 + (vert * cp) ** 2), lo, hi)
    lr = lat * rad * sp
    return az, pol, rad, lr * np.cos(az), lr * np.sin(az), vert * rad * cp


def positions(prob: OracleProblem, C: np.ndarray) -> np.ndarray:
    """(3, n, m1) coefficients -> (3, n, S) sampled positions (assembly.py:277-279)."""
    return C @ prob.W.T


def pair_diffs(prob: OracleProblem, pos: np.ndarray) -> np.ndarray:
    """(3, P, S) differences p_i - p_j, i < j lexicographic (assembly.py:281-283)."""
    return pos[:, prob.pair_i, :] - pos[:, prob.pair_j, :]


def transpose_apply(prob: OracleProblem, v_pair, v_ws) -> np.ndarray:
    """F^T on per-block values -> (3, n, m1) (assembly.py:296-303)."""
    return (np.einsum("pn,apt->ant", prob.incidence, v_pair) + v_ws) @ prob.W


def apply_F(prob: OracleProblem, xi) -> np.ndarray:
    """F xi in the flat layout [D_x; P_x; D_y; P_y; D_z; P_z] (assembly.py:1-20, 285-294)."""
    pos = positions(prob, np.asarray(xi, dtype=float).reshape(3, prob.n, prob.m1))
    d = pair_diffs(prob, pos)
    return np.concatenate([np.concatenate([d[ax].ravel(), pos[ax].ravel()]) for ax in range(3)])


def transpose_flat(prob: OracleProblem, values) -> np.ndarray:
    """F^T v for a flat stacked vector (assembly.py:305-310)."""
    P, S, n = prob.pair_i.size, prob.samples, prob.n
    v = np.asarray(values, dtype=float).reshape(3, P * S + n * S)
    return transpose_apply(prob, v[:, :P * S].reshape(3, P, S), v[:, P * S:].reshape(3, n, S)).ravel()


def spherical_rhs(prob: OracleProblem, az_p, pol_p, rad_p, az_w, pol_w, rad_w) -> np.ndarray:
    """Flat target vector e from spherical variables (assembly.py:368-408)."""
    lr = prob.lat * rad_p * np.sin(pol_p)
    pair = np.stack([lr * np.cos(az_p), lr * np.sin(az_p), prob.vert * rad_p * np.cos(pol_p)])
    lw = prob.ws_lat * rad_w * np.sin(pol_w)
    ws = np.stack([lw * np.cos(az_w), lw * np.sin(az_w), prob.ws_vert * rad_w * np.cos(pol_w)])
    ws = ws + prob.center[:, None, None]
    return np.concatenate([np.concatenate([pair[ax].ravel(), ws[ax].ravel()]) for ax in range(3)])


def project_boundary(prob: OracleProblem, xi) -> np.ndarray:
    """xi - A^T (A A^T)^{-1} (A xi - b) per robot and axis (projection.py:11-25)."""
    C = np.asarray(xi, dtype=float).reshape(3, prob.n, prob.m1)
    B = prob.endpoint
    res = np.einsum("ank,ck->anc", C, B) - prob.rhs
    y = scipy.linalg.cho_solve(scipy.linalg.cho_factor(B @ B.T), res.reshape(-1, 6).T)
    return (C - (y.T @ B).reshape(C.shape)).ravel()


class OracleSingularKKT(RuntimeError):
    """Endpoint residual above tol_eq after refinement (assembly.py:213-217)."""


def kkt_matrix(prob: OracleProblem, rho: float) -> np.ndarray:
    """Per-axis saddle matrix [[I + rho kron(inc^T inc + I, W^T W), A^T], [A, 0]] (assembly.py:164-177)."""
    n, m1 = prob.n, prob.m1
    Q = rho * np.kron(prob.incidence.T @ prob.incidence + np.eye(n), prob.W.T @ prob.W)
    Q[np.diag_indices_from(Q)] += 1.0
    A = np.kron(np.eye(n), prob.endpoint)
    K = np.zeros((n * m1 + 6 * n,) * 2)
    K[:n * m1, :n * m1] = Q
    K[:n * m1, n * m1:] = A.T
    K[n * m1:, :n * m1] = A
    return K


def kkt_solve(prob: OracleProblem, rho: float, eta_axes: np.ndarray, tol_eq: float) -> np.ndarray:
    """LU solve of the saddle system for all three axes, with the reference's
    refinement loop and SingularKKT check (assembly.py:186-219)."""
    key = float(rho)
    if key not in prob._kkt:
        K = kkt_matrix(prob, rho)
        prob._kkt[key] = (K, scipy.linalg.lu_factor(K))
    K, lu = prob._kkt[key]
    nc = prob.n * prob.m1
    rhs = np.empty((K.shape[0], 3))
    rhs[:nc] = eta_axes.reshape(3, nc).T
    rhs[nc:] = prob.rhs.reshape(3, -1).T

    def eq_err(sol):
        return float(np.abs(K[nc:] @ sol - rhs[nc:]).max())

    sol = scipy.linalg.lu_solve(lu, rhs)
    err = eq_err(sol)
    for _ in range(4):
        if err <= tol_eq:
            break
        sol = sol + scipy.linalg.lu_solve(lu, rhs - K @ sol)
        new = eq_err(sol)
        if new >= err:
            err = new
            break
        err = new
    if err > tol_eq:
        raise OracleSingularKKT(f"endpoint conditions missed by {err:.3e} after refinement "
                                f"(tolerance {tol_eq:.3e})")
    return sol[:nc].T.reshape(3, prob.n, prob.m1)


def multiplier_update(prob: OracleProblem, lam, xi, e_vec, rho) -> np.ndarray:
    """lam - rho F^T (F xi - e) (solver.py:186-199)."""
    return np.asarray(lam, dtype=float).ravel() - rho * transpose_flat(prob, apply_F(prob, xi) - e_vec)


def coefficient_step(prob: OracleProblem, xi_bar, e_vec, lam, rho, tol_eq=1e-8) -> np.ndarray:
    """Equality-constrained QP step with rhs rho F^T e + lam + xi_bar (solver.py:202-221)."""
    eta = rho * transpose_flat(prob, e_vec) + np.asarray(lam, float).ravel() + np.asarray(xi_bar, float).ravel()
    return kkt_solve(prob, rho, eta.reshape(3, -1), tol_eq).ravel()


# --------------------------------------------------------------------------- solve
@dataclass
class OracleResult:
    coeffs: np.ndarray | None
    multipliers: np.ndarray | None
    residual_inf: np.ndarray
    residual_l2: np.ndarray
    iterations: int
    converged: bool
    displacement: float
    svars: tuple | None = None     # (pair az, pol, rad, ws az, pol, rad) of the last iteration
    error: str | None = None


def solve(prob: OracleProblem, xi_bar, xi0=None, lam0=None, rho=1.0, max_iters=200,
          tol_residual=1e-3, tol_eq=1e-8, early_stop=True) -> OracleResult:
    """One SF solve; the loop of ``solver.py:286-359``.

    Default start: boundary projection of the proposal, zero multipliers
    (solver.py:264-284).  Each iteration: spherical step on the current
    positions (315), multiplier step (319-321), eta (323-327), KKT solve
    (328), residual of new positions against the targets of this iteration
    (330-342), early stop (343-345).
    """
    xb = np.asarray(xi_bar, dtype=float).ravel()
    if xb.size != prob.dim:
        raise ValueError(f"proposal has length {xb.size}, expected {prob.dim}")
    if xi0 is None:
        C = project_boundary(prob, xb).reshape(3, prob.n, prob.m1)
        lam = np.zeros((3, prob.n, prob.m1))
    else:
        C = np.asarray(xi0, dtype=float).reshape(3, prob.n, prob.m1).copy()
        lam = np.asarray(lam0, dtype=float).reshape(3, prob.n, prob.m1).copy()
    xb3 = xb.reshape(3, prob.n, prob.m1)
    ctr = prob.center[:, None, None]

    pos = positions(prob, C)
    d = pair_diffs(prob, pos)
    rel = pos - ctr
    inf_h = np.empty(max_iters)
    l2_h = np.empty(max_iters)
    its = 0
    sv = None
    try:
        for k in range(max_iters):
            pa, pp, pr, ptx, pty, ptz = spherical_project(
                d[0].ravel(), d[1].ravel(), d[2].ravel(), prob.lat, prob.vert, 1.0, np.inf)
            wa, wp, wr, wtx, wty, wtz = spherical_project(
                rel[0].ravel(), rel[1].ravel(), rel[2].ravel(), prob.ws_lat, prob.ws_vert, 0.0, 1.0)
            sv = (pa.reshape(d.shape[1:]), pp.reshape(d.shape[1:]), pr.reshape(d.shape[1:]),
                  wa.reshape(rel.shape[1:]), wp.reshape(rel.shape[1:]), wr.reshape(rel.shape[1:]))
            pt = np.stack([ptx.reshape(d.shape[1:]), pty.reshape(d.shape[1:]), ptz.reshape(d.shape[1:])])
            wt = np.stack([wtx.reshape(rel.shape[1:]), wty.reshape(rel.shape[1:]), wtz.reshape(rel.shape[1:])])
            lam = lam - rho * transpose_apply(prob, d - pt, rel - wt)
            eta = rho * transpose_apply(prob, pt, wt + ctr) + lam + xb3
            C = kkt_solve(prob, rho, eta.reshape(3, -1), tol_eq)
            pos = positions(prob, C)
            d = pair_diffs(prob, pos)
            rel = pos - ctr
            rp = d - pt
            rw = rel - wt
            sq = float(np.vdot(rp, rp) + np.vdot(rw, rw))
            inf = max(float(np.abs(rp).max()) if rp.size else 0.0, float(np.abs(rw).max()))
            inf_h[k] = inf
            l2_h[k] = np.sqrt(sq)
            its = k + 1
            if early_stop and inf <= tol_residual:
                break
    except OracleSingularKKT as exc:
        return OracleResult(None, None, np.empty(0), np.empty(0), 0, False, float("nan"),
                            error=f"SingularKKT: {exc}")
    coeffs = C.ravel().copy()
    return OracleResult(
        coeffs=coeffs, multipliers=lam.ravel().copy(),
        residual_inf=inf_h[:its].copy(), residual_l2=l2_h[:its].copy(),
        iterations=its, converged=bool(inf_h[its - 1] <= tol_residual),
        displacement=float(np.linalg.norm(coeffs - xb)), svars=sv,
    )


# --------------------------------------------------------------------------- verdict
@dataclass
class OracleVerdict:
    ok: bool
    pair_margin_min: float
    workspace_margin_max: float
    pair_violation_count: int
    workspace_violation_count: int


def check_constraints(prob: OracleProblem, coeffs, tol: float = 1e-3) -> OracleVerdict:
    """Original (non-reformulated) constraint check on the sampled trajectory.

    Follows ``basis.py:149-160`` (positions = C W^T) and
    ``assembly.py:437-487`` with the margins of ``problem.py:113-137``.
    """
    C = np.asarray(coeffs, dtype=float).reshape(3, prob.n, prob.m1)
    pos = np.moveaxis(np.einsum("ank,tk->ant", C, prob.W), 0, -1)      # (n, S, 3)
    dw = pos - prob.center
    wm = (dw[..., 0] ** 2 + dw[..., 1] ** 2) / prob.ws_lat ** 2 + dw[..., 2] ** 2 / prob.ws_vert ** 2 - 1.0
    n_ws = int((wm > tol).sum())
    pmin, n_pair = np.inf, 0
    if prob.n > 1:
        ii, jj = np.triu_indices(prob.n, k=1)
        dd = pos[ii] - pos[jj]
        pm = (dd[..., 0] ** 2 + dd[..., 1] ** 2) / prob.lat ** 2 + dd[..., 2] ** 2 / prob.vert ** 2 - 1.0
        pmin = float(pm.min())
        n_pair = int((pm < -tol).sum())
    return OracleVerdict(n_pair == 0 and n_ws == 0, pmin, float(wm.max()), n_pair, n_ws)


def feasible(prob: OracleProblem, res: OracleResult, tol: float = 1e-3) -> bool:
    """converged and passes the original constraints (metrics.py:57-69)."""
    return bool(res.converged and res.coeffs is not None and check_constraints(prob, res.coeffs, tol).ok)


def mean_pairwise_cosine(vectors) -> float:
    """Mean cosine over all unordered pairs, the reference's Gram-matrix formula (metrics.py:83-99)."""
    V = np.asarray(vectors, dtype=float)
    if V.ndim != 2:
        V = V.reshape(len(V), -1)
    norms = np.linalg.norm(V, axis=1)
    if np.any(norms == 0.0):
        return float("nan")
    U = V / norms[:, None]
    G = U @ U.T
    idx = np.triu_indices(V.shape[0], k=1)
    return float(G[idx].mean())


def diversity_cosine(position_sets, center: bool = True) -> float:
    """metrics.py:102-115 on a list of (n, S, 3) position arrays."""
    V = np.stack([np.asarray(p, dtype=float).ravel() for p in position_sets])
    if center:
        V = V - V.mean(axis=0)
    return mean_pairwise_cosine(V)
