"""One-time FP64 host precompute of the device constants.

The reference factors the full per-axis saddle system
``[[I + rho kron(inc^T inc + I, G), A^T], [A, 0]]`` (size 17n at degree 10)
with dense LU once per rho and solves it every iteration
(``assembly.py:154-219``).  Its robot-space block ``L = inc^T inc + I``
equals ``(n+1) I - 1 1^T``: eigenvalue 1 on the swarm mean and ``n+1`` on
every deviation from it.  ``A = kron(I_n, B)`` commutes with that split, so
the 17n system decouples exactly into

* one "mean" KKT ``[[I + rho G, B^T], [B, 0]]`` (17 x 17), and
* one "deviation" KKT ``[[I + rho (n+1) G, B^T], [B, 0]]`` shared by all robots,

with ``xi_i = Km11 eta_bar + Kd11 (eta_i - eta_bar) + cconst_i``.  Writing the
right-hand side through ``F^T e = F^T F xi_k - F^T r`` (the residual
identity) gives the per-iteration update the kernel runs::

    lam' = lam - rho * (R @ W)                   R: scattered residual (time domain)
    u    = 2 lam' - lam + xi_bar
    xi_i = Mm C_bar + Km11 u_bar + Md (C_i - C_bar) + Kd11 (u_i - u_bar) + cconst_i

with ``Mm = rho Km11 G`` and ``Md = rho (n+1) Kd11 G``.  This module builds those
11x11 blocks plus the boundary projector ``B^T (B B^T)^-1`` used for the
default start (``projection.py:11-25``).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .basis import BasisMatrices
from .errors import DimensionMismatch, RankDeficient, SingularKKT

CONDITIONS = 6   # p0 v0 a0 pT vT aT


def endpoint_rows(basis: BasisMatrices) -> np.ndarray:
    """The 6 x m1 block sampling (p0, v0, a0, pT, vT, aT) (assembly.py:42-53)."""
    return np.stack([basis.value[0], basis.velocity[0], basis.acceleration[0],
                     basis.value[-1], basis.velocity[-1], basis.acceleration[-1]])


def endpoint_rhs(problem) -> np.ndarray:
    """(3, n, 6) right-hand side of the endpoint system (assembly.py:120-130)."""
    rhs = np.empty((3, problem.n, CONDITIONS))
    for i, rb in enumerate(problem.boundary):
        rhs[:, i, :] = np.stack([rb.start.position, rb.start.velocity, rb.start.acceleration,
                                 rb.goal.position, rb.goal.velocity, rb.goal.acceleration], axis=1)
    return rhs


def _kkt_inverse(H: np.ndarray, B: np.ndarray) -> np.ndarray:
    m1 = H.shape[0]
    K = np.zeros((m1 + CONDITIONS, m1 + CONDITIONS))
    K[:m1, :m1] = H
    K[:m1, m1:] = B.T
    K[m1:, :m1] = B
    try:
        return np.linalg.solve(K, np.eye(K.shape[0]))
    except np.linalg.LinAlgError as exc:
        raise SingularKKT("saddle system factorization failed") from exc


@dataclass(frozen=True)
class EqualitySystem:
    """Endpoint conditions: shared 6 x m1 block, (3, n, 6) rhs, projector B^T (B B^T)^-1."""

    n: int
    degree: int
    block: np.ndarray
    rhs_axes: np.ndarray
    projector: np.ndarray      # (m1, 6)

    @property
    def coeff_dim(self) -> int:
        return 3 * self.n * (self.degree + 1)

    @property
    def rhs(self) -> np.ndarray:
        return self.rhs_axes.ravel()

    def apply(self, coeffs) -> np.ndarray:
        C = np.asarray(coeffs, dtype=float).reshape(3, self.n, self.degree + 1)
        return np.einsum("ank,ck->anc", C, self.block).ravel()

    def residual(self, coeffs) -> np.ndarray:
        return self.apply(coeffs) - self.rhs

    def matrix(self) -> np.ndarray:
        return np.kron(np.eye(3 * self.n), self.block)


def build_equality(problem, basis: BasisMatrices) -> EqualitySystem:
    if basis.samples != problem.horizon_samples:
        raise DimensionMismatch(f"basis has {basis.samples} samples, problem expects "
                                f"{problem.horizon_samples}")
    B = endpoint_rows(basis)
    gram = B @ B.T
    try:
        np.linalg.cholesky(gram)
    except np.linalg.LinAlgError as exc:
        raise RankDeficient("endpoint condition rows are linearly dependent; "
                            f"degree {basis.degree} with duration {basis.duration}") from exc
    return EqualitySystem(problem.n, basis.degree, B, endpoint_rhs(problem),
                          B.T @ np.linalg.inv(gram))


@dataclass(frozen=True)
class DeviceConstants:
    """FP64 constants uploaded once per (problem, degree, rho); see module doc."""

    n: int
    samples: int
    m1: int
    rho: float
    lat: float
    vert: float
    ws_lat: float
    ws_vert: float
    center: np.ndarray        # (3,)
    W: np.ndarray             # (S, m1)
    Wd: np.ndarray            # (S, m1)
    Wdd: np.ndarray           # (S, m1)
    B: np.ndarray             # (6, m1)
    rhs: np.ndarray           # (3, n, 6)
    PBt: np.ndarray           # (m1, 6)   boundary projector B^T (B B^T)^-1
    Km11: np.ndarray          # (m1, m1)
    Kd11: np.ndarray
    Mm: np.ndarray            # rho Km11 G
    Md: np.ndarray            # rho (n+1) Kd11 G
    cconst: np.ndarray        # (3, n, m1)


def _projector(equality, B: np.ndarray) -> np.ndarray:
    """B^T (B B^T)^-1 (m1 x 6).  This package's EqualitySystem carries it; the reference's
    (``assembly.py:56-70``: block, rhs_axes and a Cholesky factor of B B^T) does not, so derive it."""
    proj = getattr(equality, "projector", None)
    if proj is not None:
        return proj
    return B.T @ np.linalg.inv(B @ B.T)


def device_constants(problem, basis: BasisMatrices, equality: EqualitySystem, rho: float) -> DeviceConstants:
    """FP64 constants of one (problem, degree, rho).  ``problem``, ``basis`` and ``equality`` may be this
    package's objects or the reference's (``swarmfilter.SafetyFilter``'s problem / basis / equality: same
    attribute names, ``problem.py:28-104``, ``basis.py:73-88``, ``assembly.py:56-70``)."""
    if not rho >= 0:
        raise ValueError(f"penalty weight must be nonnegative, got {rho}")
    n, m1 = problem.n, basis.degree + 1
    W = basis.value
    G = W.T @ W
    B = equality.block
    eye = np.eye(m1)
    Km = _kkt_inverse(eye + rho * G, B)
    Kd = _kkt_inverse(eye + rho * (n + 1) * G, B)
    Km11, Km12 = Km[:m1, :m1], Km[:m1, m1:]
    Kd11, Kd12 = Kd[:m1, :m1], Kd[:m1, m1:]
    rhs = equality.rhs_axes
    bbar = rhs.mean(axis=1, keepdims=True)                       # (3, 1, 6)
    cconst = (bbar @ Km12.T) + ((rhs - bbar) @ Kd12.T)            # (3, n, m1)
    ws = problem.workspace
    return DeviceConstants(
        n=n, samples=basis.samples, m1=m1, rho=float(rho),
        lat=float(problem.shape.lateral), vert=float(problem.shape.vertical),
        ws_lat=float(ws.lateral), ws_vert=float(ws.vertical),
        center=np.asarray(ws.center, dtype=float).copy(),
        W=np.ascontiguousarray(W), Wd=np.ascontiguousarray(basis.velocity),
        Wdd=np.ascontiguousarray(basis.acceleration),
        B=np.ascontiguousarray(B), rhs=np.ascontiguousarray(rhs),
        PBt=np.ascontiguousarray(_projector(equality, B)),
        Km11=np.ascontiguousarray(Km11), Kd11=np.ascontiguousarray(Kd11),
        Mm=np.ascontiguousarray(rho * Km11 @ G), Md=np.ascontiguousarray(rho * (n + 1) * Kd11 @ G),
        cconst=np.ascontiguousarray(cconst),
    )


def decoupled_step_host(k: DeviceConstants, C, lam_new, lam, xi_bar) -> np.ndarray:
    """FP64 numpy statement of the device xi-step (used by CPU tests of the precompute)."""
    C = np.asarray(C, float).reshape(3, k.n, k.m1)
    u = (2.0 * np.asarray(lam_new, float) - np.asarray(lam, float) + np.asarray(xi_bar, float)).reshape(3, k.n, k.m1)
    Cb = C.mean(axis=1, keepdims=True)
    ub = u.mean(axis=1, keepdims=True)
    out = Cb @ k.Mm.T + ub @ k.Km11.T + (C - Cb) @ k.Md.T + (u - ub) @ k.Kd11.T + k.cconst
    return out.ravel()
