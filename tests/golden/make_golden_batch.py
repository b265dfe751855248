"""Freeze the REAL reference's outputs on whole benchmark batches (build container only).

    python tests/golden/make_golden_batch.py cfg2        # all 1000 config-2 bench proposals
    python tests/golden/make_golden_batch.py ws_tight    # converged-but-violating workspace case
    python tests/golden/make_golden_batch.py cfg3 cfg4   # early-stop subsets at n = 32 / 64
    python tests/golden/make_golden_batch.py fuzz        # 64 random scenarios x 8 proposals, early stop
    python tests/golden/make_golden_batch.py fuzz_large  # 24 random 17..64-robot scenarios x 4 proposals

Like ``make_golden.py`` this builds the reference's own Cython kernel in a
scratch copy of ``/root/reference/pkg`` and imports ``swarmfilter`` from it
(``active_backend() == 'compiled'``); nothing from the reference enters the
repo except the numbers it produced.  Each proposal is solved by
``SafetyFilter.solve`` (``solver.py:286-359``) in a process pool with BLAS
pinned to one thread, then checked by ``metrics.feasible_results``
(``metrics.py:57-69``) and ``check_original_constraints``
(``assembly.py:437-487``) -- the exact numerator of the headline metric.

Stored per sample: iterations, converged, feasible, the reference's worst
margins and violation counts, the first 8 worst-first violation entries, the
full ``res_inf`` history (float64, NaN padded: it is what decides iteration
counts, and what classifies a GPU count flip as borderline) and
the displacement.  Coefficients and multipliers are stored for a subset.
Proposals are not stored: both sides regenerate them from the reference
Gaussian sampler (seed 0) -- a SHA-256 of the float64 bytes pins them.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

os.environ["OPENBLAS_NUM_THREADS"] = "1"
os.environ["OMP_NUM_THREADS"] = "1"
os.environ["MKL_NUM_THREADS"] = "1"

import numpy as np  # noqa: E402

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(REPO))

LISTED = 8   # worst-first violation entries stored per kind

_W = {}


def _init(doc, degree, cfg):
    from make_golden import import_reference
    sfm = import_reference()
    prob = sfm.load_problem(doc) if isinstance(doc, dict) else doc
    _W["sfm"] = sfm
    _W["prob"] = prob
    _W["filt"] = sfm.SafetyFilter(prob, degree=degree, config=sfm.SolverConfig(**cfg))


def _solve_one(args):
    idx, x = args
    sfm, prob, filt = _W["sfm"], _W["prob"], _W["filt"]
    t0 = time.perf_counter()
    r = filt.solve(x)
    dt = time.perf_counter() - t0
    traj = sfm.coeffs_to_trajectory(r.coeffs, filt.basis, prob.n)
    rep = sfm.check_original_constraints(traj, prob, tol=1e-3)
    feas = bool(r.converged and rep.ok)
    # feasible_results is the headline's own definition: check it agrees
    assert feas == (len(sfm.metrics.feasible_results([r], prob)) == 1)
    return (idx, r.iterations, bool(r.converged), feas, float(rep.pair_margin_min),
            float(rep.workspace_margin_max), rep.pair_violation_count, rep.workspace_violation_count,
            [list(v) for v in rep.pair_violations[:LISTED]], [list(v) for v in rep.workspace_violations[:LISTED]],
            np.asarray(r.residual_inf), np.asarray(r.residual_l2), float(r.displacement),
            np.asarray(r.coeffs), np.asarray(r.multipliers), dt)


def run_batch(name, doc, proposals, degree=10, keep_coeffs=64, procs=None, select=None, save=True, **cfg):
    import multiprocessing as mp
    B = len(proposals)
    maxit = cfg.get("max_iters", 200)
    procs = procs or os.cpu_count() or 1
    out = {
        "iterations": np.zeros(B, np.int32), "converged": np.zeros(B, bool), "feasible": np.zeros(B, bool),
        "pair_margin_min": np.full(B, np.nan), "ws_margin_max": np.full(B, np.nan),
        "pair_viol": np.zeros(B, np.int32), "ws_viol": np.zeros(B, np.int32),
        "pair_list": np.full((B, LISTED, 4), np.nan), "ws_list": np.full((B, LISTED, 3), np.nan),
        "res_inf": np.full((B, maxit), np.nan), "res_l2_last": np.full(B, np.nan),
        "displacement": np.full(B, np.nan),
        "coeffs_subset": np.full((min(B, keep_coeffs), len(proposals[0])), np.nan),
        "multipliers_subset": np.full((min(B, keep_coeffs), len(proposals[0])), np.nan),
    }
    t0 = time.perf_counter()
    cpu = 0.0
    with mp.get_context("fork").Pool(procs, initializer=_init, initargs=(doc, degree, cfg)) as pool:
        for k, row in enumerate(pool.imap_unordered(_solve_one, list(enumerate(proposals)), chunksize=1)):
            (i, its, conv, feas, pmin, wmax, pv, wv, pl, wl, rinf, rl2, disp, co, mu, dt) = row
            cpu += dt
            out["iterations"][i] = its
            out["converged"][i] = conv
            out["feasible"][i] = feas
            out["pair_margin_min"][i] = pmin
            out["ws_margin_max"][i] = wmax
            out["pair_viol"][i] = pv
            out["ws_viol"][i] = wv
            for j, v in enumerate(pl):
                out["pair_list"][i, j] = v
            for j, v in enumerate(wl):
                out["ws_list"][i, j] = v
            out["res_inf"][i, :its] = rinf
            out["res_l2_last"][i] = rl2[-1]
            out["displacement"][i] = disp
            if i < keep_coeffs:
                out["coeffs_subset"][i] = co
                out["multipliers_subset"][i] = mu
            if (k + 1) % 50 == 0:
                print(f"  {name}: {k + 1}/{B} ({time.perf_counter() - t0:.0f} s)", flush=True)
    wall = time.perf_counter() - t0
    sha = hashlib.sha256(np.ascontiguousarray(np.asarray(proposals, dtype=np.float64)).tobytes()).hexdigest()
    meta = {"name": name, "problem": doc, "degree": degree, "config": cfg, "batch": B,
            "proposals_sha256": sha, "reference_backend": "compiled", "wall_s": wall, "cpu_s": cpu,
            "procs": procs, "sample_iterations": int(out["iterations"].sum())}
    if select is not None:   # rows `indices` of a `batch`-sample draw (seed 0) of bench.py's batch
        meta["select"] = select
    if not save:
        return out, meta
    np.savez_compressed(HERE / f"{name}.npz", meta=np.array(json.dumps(meta)), **out)
    print(f"{name}: B={B} iterations {out['iterations'].min()}..{out['iterations'].max()} "
          f"(mean {out['iterations'].mean():.1f}) converged {out['converged'].sum()} "
          f"feasible {out['feasible'].sum()} ws_viol>0 {(out['ws_viol'] > 0).sum()} "
          f"pair_viol>0 {(out['pair_viol'] > 0).sum()}  wall {wall:.0f} s, {cpu / max(1, meta['sample_iterations']) * 1e3:.2f} ms/SI",
          flush=True)


def proposals_for(doc, batch, seed=0, degree=10, spread=0.25):
    """The bench's inputs: this repo's sampler (== the reference sampler, test_host.py pins it)."""
    from paper_2501_19042_b200 import load_problem, sample_proposals
    from paper_2501_19042_b200.basis import build_basis
    prob = load_problem(doc)
    basis = build_basis(prob.duration, degree=degree, samples=prob.horizon_samples)
    return sample_proposals(prob, basis, batch, seed=seed, spread=spread).proposals


def ws_tight_doc():
    """6 robots in a workspace barely larger than their start/goal sets; loose tol_residual.

    With tol_residual = 0.05 the SF stops while some positions still poke out of
    the workspace spheroid by more than the verdict's 1e-3: converged-but-
    infeasible on the *workspace* branch of ``check_original_constraints``.
    """
    starts = [(2.2, 0.0, 1.0), (-2.2, 0.3, 1.2), (0.0, 2.1, 0.8), (0.2, -2.2, 1.1), (1.4, 1.5, 1.6), (-1.5, -1.4, 0.5)]
    goals = [(-2.2, 0.2, 1.1), (2.2, -0.1, 0.9), (0.1, -2.1, 1.2), (-0.2, 2.2, 0.8), (-1.5, -1.4, 0.6), (1.4, 1.5, 1.5)]
    return {"n": 6, "H": 60, "T": 6.0, "a": 0.6, "b": 0.4,
            "workspace": {"center": [0.0, 0.0, 1.0], "a_w": 2.6, "b_w": 1.2},
            "boundary": [{"start": {"p": list(s)}, "goal": {"p": list(g)}} for s, g in zip(starts, goals)]}


FUZZ_MAXIT = 300


def fuzz_cases_large(count=24, seed=4242):
    """Random scenarios for the large-swarm fuzz fixture: 17..64 robots (the two-lane K1 slot and K1L, FP64 K1L
    for strict), horizons 20..100, degrees 7..15, rho and tol_residual varied; 4 proposals each."""
    rng = np.random.default_rng(seed)
    cases = []
    for c in range(count):
        n = int(rng.integers(17, 33)) if c % 2 == 0 else int(rng.integers(33, 65))
        H = int(rng.choice([20, 40, 60, 100]))
        cases.append({"n": n, "H": H, "scenario_seed": int(rng.integers(0, 10000)),
                      "degree": int(rng.integers(7, 16)), "rho": float(rng.choice([0.5, 1.0, 2.0])),
                      "tol_residual": float(rng.choice([1e-3, 3e-3, 1e-2])),
                      "spread": float(rng.choice([0.25, 0.6])), "seed": int(rng.integers(0, 1000)), "batch": 4})
    return cases


def fuzz_cases(count=64, seed=2026):
    """Random scenarios for the early-stop fuzz fixture: robots 2..40 (every K1 template, the tensor-core
    n = 16 slot, the two-lane n = 17..32 slot and K1L), horizons 20..127, degrees 7..15, rho, tol_residual and
    proposal spread varied; 8 proposals each."""
    from paper_2501_19042_b200.scenarios import random_swarm_doc
    rng = np.random.default_rng(seed)
    cases = []
    for c in range(count):
        u = rng.random()
        if u < 0.55:
            n = int(rng.choice([2, 3, 4, 5, 6, 7, 8, 9, 11, 12]))
            H = int(rng.choice([20, 40, 60, 100, 120]))
        elif u < 0.85:
            n = int(rng.choice([13, 14, 15, 16]))
            H = int(rng.choice([40, 60, 96, 100, 110, 127]))
        elif u < 0.95:
            n = int(rng.integers(17, 33))
            H = int(rng.choice([20, 30, 40]))
        else:
            n = int(rng.integers(33, 41))
            H = int(rng.choice([20, 30]))
        cases.append({"n": n, "H": H, "scenario_seed": int(rng.integers(0, 10000)),
                      "degree": int(rng.integers(7, 16)), "rho": float(rng.choice([0.5, 1.0, 2.0])),
                      "tol_residual": float(rng.choice([1e-3, 1e-3, 3e-3, 1e-2])),
                      "spread": float(rng.choice([0.25, 0.6, 1.0])), "seed": int(rng.integers(0, 1000)), "batch": 8})
    return cases


def fuzz_doc(case):
    from paper_2501_19042_b200.scenarios import random_swarm_doc
    return random_swarm_doc(case["n"], case["H"], case["scenario_seed"])


def run_fuzz(name="batch_fuzz", count=64, seed=2026, large=False):
    """One fixture of many small random scenarios (early stop on), concatenated; meta["cases"] says how each
    slice was made (problem, degree, solver config, proposal seed / spread, SHA-256 of the proposals)."""
    parts, cases = [], []
    off = 0
    todo = fuzz_cases_large(count, seed) if large else fuzz_cases(count, seed)
    dmax = max(3 * c["n"] * (c["degree"] + 1) for c in todo)   # subset rows NaN-padded to the widest case
    for case in todo:
        doc = fuzz_doc(case)
        x = proposals_for(doc, case["batch"], seed=case["seed"], degree=case["degree"], spread=case["spread"])
        out, meta = run_batch(f"{name}[{len(cases)}]", doc, x, degree=case["degree"], keep_coeffs=case["batch"],
                              save=False, max_iters=FUZZ_MAXIT, rho=case["rho"], tol_residual=case["tol_residual"])
        out["tol"] = np.full(case["batch"], case["tol_residual"])
        for k in ("coeffs_subset", "multipliers_subset"):
            pad = np.full((case["batch"], dmax), np.nan)
            pad[:, :out[k].shape[1]] = out[k]
            out[k] = pad
        parts.append(out)
        cases.append({**case, "problem": doc, "offset": off, "proposals_sha256": meta["proposals_sha256"],
                      "config": meta["config"]})
        off += case["batch"]
        print(f"  case {len(cases) - 1}: n={case['n']} H={case['H']} deg={case['degree']} rho={case['rho']} "
              f"tol={case['tol_residual']} its {out['iterations'].tolist()} feasible {int(out['feasible'].sum())}",
              flush=True)
    full = {k: np.concatenate([p[k] for p in parts]) for k in parts[0]}
    meta = {"name": name, "cases": cases, "batch": off, "reference_backend": "compiled", "degree": None,
            "config": {"max_iters": FUZZ_MAXIT}}
    np.savez_compressed(HERE / f"{name}.npz", meta=np.array(json.dumps(meta)), **full)
    it = full["iterations"]
    print(f"{name}: {len(cases)} scenarios, {off} samples, iterations {it.min()}..{it.max()} "
          f"converged {full['converged'].sum()} feasible {full['feasible'].sum()} "
          f"pair_viol>0 {(full['pair_viol'] > 0).sum()} ws_viol>0 {(full['ws_viol'] > 0).sum()}", flush=True)


def main(argv):
    from make_golden import import_reference
    from paper_2501_19042_b200.scenarios import config_doc
    import_reference()   # build the scratch copy once, before the pool forks
    for which in argv or ["cfg2"]:
        if which == "cfg2":
            doc = config_doc(2)
            run_batch("batch_cfg2", doc, proposals_for(doc, 1000), max_iters=500)
        elif which == "ws_tight":
            doc = ws_tight_doc()
            props = proposals_for(doc, 48, seed=3, spread=3.0)
            run_batch("batch_ws_tight", doc, props, keep_coeffs=48, max_iters=300, tol_residual=0.05)
        elif which == "cfg3":   # the first 16 proposals of bench.py --config 3's batch
            doc = config_doc(3)
            run_batch("batch_cfg3", doc, proposals_for(doc, 16), keep_coeffs=16, max_iters=500)
        elif which == "cfg4":   # the first 8 proposals of bench.py --config 4's batch (all reach the cap)
            doc = config_doc(4)
            run_batch("batch_cfg4", doc, proposals_for(doc, 8), keep_coeffs=8, max_iters=1000)
        elif which == "cfg4e":  # 8 proposals of the config-4 batch that stop early (chosen from a GPU run of
            doc = config_doc(4)  # the first 1024: 1 to 671 iterations, one converged-but-infeasible)
            idx = [789, 315, 566, 526, 448, 513, 938, 681]
            run_batch("batch_cfg4e", doc, proposals_for(doc, 1024)[idx], keep_coeffs=8, max_iters=1000,
                      select={"batch": 1024, "indices": idx})
        elif which == "fuzz":   # random small scenarios with early stop (every kernel family)
            run_fuzz()
        elif which == "fuzz_large":   # random 17..64-robot scenarios with early stop (two-lane K1, K1L)
            run_fuzz("batch_fuzz_large", count=24, seed=4242, large=True)
        else:
            raise SystemExit(f"unknown batch {which}")


if __name__ == "__main__":
    main(sys.argv[1:])
