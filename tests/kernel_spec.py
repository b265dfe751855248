"""numpy statement of the algorithm the CUDA kernel runs (test tool, CPU only).

Used by CPU tests to validate the kernel's reformulation against the oracle
before any GPU time is spent, and to pin the precision recipe:

* decoupled FP64 xi-step (precompute.py docstring),
* residual identity F^T e = F^T F xi - F^T r,
* trig-free spherical projection t = s d with s = clamp(r)/r,
  falling back to the reference trig formula in FP64 whenever a component of
  d is exactly zero,
* pair/workspace term work, positions and the W^T projection in ``term``
  precision (float32 "lean" or float64 "strict"), state in FP64.

The pass structure is the kernel's: pass k builds targets from positions k
and, for k >= 1, the exit residual of iteration k-1 against the targets of
iteration k-1 recomputed from positions k-1.
"""
from __future__ import annotations

import numpy as np


def fallback_project(dx, dy, dz, lat, vert, lo, hi):
    """Reference trig formula (kernels/reference.py:13-48) in FP64."""
    az = np.arctan2(dy, dx)
    planar = np.hypot(dx, dy)
    pol = np.arctan2(planar / lat, dz / vert)
    pol = np.where((planar == 0.0) & (dz == 0.0), 0.5 * np.pi, pol)
    sp, cp = np.sin(pol), np.cos(pol)
    rad = np.clip((lat * sp * planar + vert * cp * dz) / ((lat * sp) ** 2 + (vert * cp) ** 2), lo, hi)
    lr = lat * rad * sp
    return lr * np.cos(az), lr * np.sin(az), vert * rad * cp


def project(d, lat, vert, lo, hi, dt):
    """Targets for difference vectors d (3, ...) in precision dt."""
    d = d.astype(dt)
    dx, dy, dz = d
    beta = dt(lat * lat / (vert * vert))
    q = dx * dx + dy * dy + (dz * beta) * dz          # = lat^2 r^2
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.sqrt(q) / dt(lat)
        s = np.clip(r, dt(lo), dt(hi)) / r
    inside = (r >= lo) & (r <= hi)
    s = np.where(inside, dt(1.0), s)
    t = (s * d).astype(dt)
    zero = (dx == 0) | (dy == 0) | (dz == 0)
    if zero.any():
        fx, fy, fz = fallback_project(dx[zero].astype(np.float64), dy[zero].astype(np.float64),
                                      dz[zero].astype(np.float64), lat, vert, lo, hi)
        t[0][zero], t[1][zero], t[2][zero] = fx, fy, fz
    return t


def spec_solve(k, xi_bar, xi0=None, lam0=None, max_iters=200, tol_residual=1e-3, early_stop=True,
               term=np.float32):
    """k: precompute.DeviceConstants.  Returns dict like the kernel outputs."""
    n, m1 = k.n, k.m1
    dt = term
    W = k.W.astype(dt)
    xb = np.asarray(xi_bar, float).reshape(3, n, m1)
    if xi0 is None:
        res = xb @ k.B.T - k.rhs
        C = xb - res @ k.PBt.T
        lam = np.zeros((3, n, m1))
    else:
        C = np.asarray(xi0, float).reshape(3, n, m1).copy()
        lam = np.asarray(lam0, float).reshape(3, n, m1).copy()
    pi, pj = np.triu_indices(n, k=1)
    ctr = k.center.astype(dt)[:, None, None]
    hist_inf, hist_l2 = [], []
    pos_old = None
    it = 0
    while True:
        pos = (C.astype(dt) @ W.T).astype(dt)               # (3, n, S)
        d = pos[:, pi, :] - pos[:, pj, :]
        rel = pos - ctr
        if pos_old is not None:
            # exit residual of iteration it-1: new positions vs targets of it-1
            do = pos_old[:, pi, :] - pos_old[:, pj, :]
            eo = project(do, k.lat, k.vert, 1.0, np.inf, dt)
            wo = project(pos_old - ctr, k.ws_lat, k.ws_vert, 0.0, 1.0, dt)
            rp = d - eo
            rw = rel - wo
            inf = max(float(np.abs(rp).max()) if rp.size else 0.0, float(np.abs(rw).max()))
            l2 = float(np.sqrt(np.sum(rp.astype(np.float64) ** 2) + np.sum(rw.astype(np.float64) ** 2)))
            hist_inf.append(inf)
            hist_l2.append(l2)
            if (early_stop and inf <= tol_residual) or it == max_iters:
                break
        e = project(d, k.lat, k.vert, 1.0, np.inf, dt)
        w = project(rel, k.ws_lat, k.ws_vert, 0.0, 1.0, dt)
        r = (d - e).astype(dt)
        acc = (rel - w).astype(dt)
        np.add.at(acc, (slice(None), pi), r)
        np.subtract.at(acc, (slice(None), pj), r)
        g = (acc @ W).astype(np.float64)
        lam_new = lam - k.rho * g
        u = 2.0 * lam_new - lam + xb
        Cb = C.mean(axis=1, keepdims=True)
        ub = u.mean(axis=1, keepdims=True)
        C = Cb @ k.Mm.T + ub @ k.Km11.T + (C - Cb) @ k.Md.T + (u - ub) @ k.Kd11.T + k.cconst
        lam = lam_new
        pos_old = pos
        it += 1
    its = len(hist_inf)
    return {"coeffs": C.ravel(), "multipliers": lam.ravel(), "res_inf": np.array(hist_inf),
            "res_l2": np.array(hist_l2), "iterations": its,
            "converged": bool(hist_inf[-1] <= tol_residual),
            "displacement": float(np.linalg.norm(C.ravel() - xb.ravel()))}
