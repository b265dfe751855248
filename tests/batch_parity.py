"""Whole-batch parity of the sm_100a solve against the REAL reference's frozen outputs.

The fixtures (``tests/golden/batch_*.npz``, made by ``make_golden_batch.py``) hold, per
sample, what the compiled reference returned on the exact headline batch: iterations,
converged, the feasible verdict (``metrics.py:57-69`` -> ``assembly.py:437-487``), its worst
margins and violation counts, the full ``res_inf`` history, and coefficients for a subset.
``compare`` regenerates the same proposals (SHA-256-pinned), runs ``solve_batched`` in the
requested precision and classifies every disagreement:

* an iteration-count flip is *borderline* when the reference's own exit residual at the first
  iteration where the two runs stop differently lies within ``band`` (relative) of
  ``tol_residual`` -- the count is decided by a residual that sits on the threshold;
* a verdict flip among samples with identical counts is *borderline* when the reference's
  deciding margin lies within ``band`` (absolute, in margin units) of the verdict threshold.

Used by ``tests/test_gpu_batch_parity.py`` (gates) and ``tools/batch_parity.py`` (report).
"""
from __future__ import annotations

import hashlib
import json

import numpy as np

from .conftest import load_golden

# how each fixture's proposals were drawn (make_golden_batch.py): batch, seed, spread
BATCHES = {"batch_cfg2": (1000, 0, 0.25), "batch_ws_tight": (48, 3, 3.0), "batch_cfg3": (16, 0, 0.25),
           "batch_cfg4": (8, 0, 0.25), "batch_cfg4e": (1024, 0, 0.25)}


def proposals(name: str, meta: dict) -> np.ndarray:
    from paper_2501_19042_b200 import load_problem, sample_proposals
    from paper_2501_19042_b200.basis import build_basis
    B, seed, spread = BATCHES[name]
    prob = load_problem(meta["problem"])
    basis = build_basis(prob.duration, degree=meta["degree"], samples=prob.horizon_samples)
    x = sample_proposals(prob, basis, B, seed=seed, spread=spread).proposals
    if "select" in meta:   # rows of a larger draw
        x = np.ascontiguousarray(x[meta["select"]["indices"]])
    sha = hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).tobytes()).hexdigest()
    assert sha == meta["proposals_sha256"], f"{name}: regenerated proposals differ from the fixture's"
    return x


def run(name: str, precision: str, **solve_kw) -> tuple[dict, dict]:
    """Solve the fixture's batch on the GPU; returns (golden, outputs as numpy)."""
    import torch

    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, load_problem
    from paper_2501_19042_b200.verdict import verdict_batched
    g = load_golden(name)
    meta = g["meta"]
    x = proposals(name, meta)
    cfg = SolverConfig(precision=precision, svars=False, **meta["config"])
    sf = SafetyFilter(load_problem(meta["problem"]), degree=meta["degree"], config=cfg)
    out = sf.solve_batched(torch.from_numpy(x).cuda(), config=cfg, **solve_kw)
    v = verdict_batched(sf.operator, out.coeffs, out.converged, tol=1e-3)
    torch.cuda.synchronize()
    o = {k: (t.cpu().numpy() if isinstance(t, torch.Tensor) else t) for k, t in vars(out).items()}
    o.update({f"v_{k}": t.cpu().numpy() for k, t in v.items()})
    return g, o


def run_fuzz(precision: str, name: str = "batch_fuzz") -> tuple[dict, dict]:
    """``batch_fuzz``: many small random scenarios (make_golden_batch.py ``fuzz``), each solved as its own batch;
    the outputs are concatenated in fixture order (coefficients NaN-padded to the widest case)."""
    import torch

    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, load_problem, sample_proposals
    from paper_2501_19042_b200.basis import build_basis
    from paper_2501_19042_b200.verdict import verdict_batched
    g = load_golden(name)
    width = g["coeffs_subset"].shape[1]
    parts = []
    for case in g["meta"]["cases"]:
        prob = load_problem(case["problem"])
        basis = build_basis(prob.duration, degree=case["degree"], samples=prob.horizon_samples)
        x = sample_proposals(prob, basis, case["batch"], seed=case["seed"], spread=case["spread"]).proposals
        sha = hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).tobytes()).hexdigest()
        assert sha == case["proposals_sha256"], f"{name}: case {case['offset']}: regenerated proposals differ"
        cfg = SolverConfig(precision=precision, svars=False, **case["config"])
        sf = SafetyFilter(prob, degree=case["degree"], config=cfg)
        out = sf.solve_batched(torch.from_numpy(x).cuda(), config=cfg)
        v = verdict_batched(sf.operator, out.coeffs, out.converged, tol=1e-3)
        torch.cuda.synchronize()
        o = {k: (t.cpu().numpy() if isinstance(t, torch.Tensor) else t) for k, t in vars(out).items()}
        o.update({f"v_{k}": t.cpu().numpy() for k, t in v.items()})
        c = np.full((case["batch"], width), np.nan)
        c[:, :o["coeffs"].shape[1]] = o["coeffs"]
        o["coeffs"] = c
        parts.append(o)
    keys = ["coeffs", "iterations", "converged", "feasible", "status", "residual_inf"] + \
        [k for k in parts[0] if k.startswith("v_")]
    return g, {k: np.concatenate([p[k] for p in parts]) for k in keys}


def compare(g: dict, o: dict, band: float) -> dict:
    """Classify every disagreement between the GPU outputs ``o`` and the golden ``g``."""
    meta = g["meta"]
    B = len(g["iterations"])
    # per-sample stopping tolerance (batch_fuzz varies it per scenario)
    tols = g["tol"] if "tol" in g else np.full(B, meta["config"].get("tol_residual", 1e-3))
    it_ref, it = g["iterations"].astype(int), o["iterations"].astype(int)
    rep = {"batch": B, "iter_equal": int((it_ref == it).sum()), "iter_flips": [], "verdict_flips": [],
           "converged_equal": int((g["converged"] == o["converged"].astype(bool)).sum()),
           "feasible_equal": int((g["feasible"] == o["feasible"].astype(bool)).sum()),
           "feasible_ref": int(g["feasible"].sum()), "feasible_gpu": int(o["feasible"].sum()),
           "status_ok": int((o["status"] == 0).sum())}
    for s in np.nonzero(it_ref != it)[0]:
        k = min(it_ref[s], it[s]) - 1           # the first iteration where exactly one run stops
        r, tol = float(g["res_inf"][s, k]), float(tols[s])
        rep["iter_flips"].append({"sample": int(s), "ref": int(it_ref[s]), "gpu": int(it[s]),
                                  "ref_res_at_split": r, "rel_to_tol": abs(r - tol) / tol,
                                  "borderline": abs(r - tol) <= band * tol})
    same = it_ref == it
    for s in np.nonzero(same & (g["feasible"] != o["feasible"].astype(bool)))[0]:
        pm, wm = float(g["pair_margin_min"][s]), float(g["ws_margin_max"][s])
        # distance of the reference's deciding margin from the verdict threshold (1e-3)
        d = min(abs(pm + 1e-3), abs(wm - 1e-3))
        rep["verdict_flips"].append({"sample": int(s), "ref": bool(g["feasible"][s]),
                                     "gpu": bool(o["feasible"][s]), "margin_dist": d,
                                     "gpu_pair_margin_min": float(o["v_pair_margin_min"][s]),
                                     "ref_pair_margin_min": pm, "borderline": d <= band})
    # margins and violation counts where both stopped at the same iterate
    pm_err = np.abs(o["v_pair_margin_min"][same] - g["pair_margin_min"][same])
    wm_err = np.abs(o["v_ws_margin_max"][same] - g["ws_margin_max"][same])
    rep["margin_err_max"] = float(max(pm_err.max(initial=0.0), wm_err.max(initial=0.0)))
    rep["viol_count_equal"] = int(((o["v_pair_viol"] == g["pair_viol"]) & (o["v_ws_viol"] == g["ws_viol"]))[same].sum())
    rep["same_iterate"] = int(same.sum())
    # coefficients on the stored subset (only where the counts agree: same iterate)
    K = g["coeffs_subset"].shape[0]
    errs = []
    for s in range(K):
        ref = g["coeffs_subset"][s]
        m = np.isfinite(ref)   # (batch_fuzz: NaN padding past the case's dimension)
        if same[s] and m.any():
            errs.append(np.abs(o["coeffs"][s][m] - ref[m]).max() / max(1.0, np.abs(ref[m]).max()))
    rep["coeff_rel_err_max"] = float(max(errs)) if errs else None
    # residual histories over the common prefix
    hist = []
    for s in range(B):
        m = min(it_ref[s], it[s])
        hr = g["res_inf"][s, :m]
        hist.append(np.max(np.abs(o["residual_inf"][s, :m] - hr) / np.maximum(hr, 1e-12)))
    rep["res_inf_rel_err_max"] = float(np.max(hist))
    rep["res_inf_rel_err_median"] = float(np.median(hist))
    rep["iter_flip_count"] = len(rep["iter_flips"])
    rep["iter_flip_nonborderline"] = sum(1 for f in rep["iter_flips"] if not f["borderline"])
    rep["verdict_flip_count"] = len(rep["verdict_flips"])
    rep["verdict_flip_nonborderline"] = sum(1 for f in rep["verdict_flips"] if not f["borderline"])
    rep["iterations_total_ref"] = int(it_ref.sum())
    rep["iterations_total_gpu"] = int(it.sum())
    return rep


def dumps(rep: dict) -> str:
    return json.dumps(rep, indent=1, default=float)
