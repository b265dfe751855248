"""Generate the golden fixtures in tests/golden/ by running the REAL reference.

Run in the build container only (it reads /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py

It copies /root/reference/pkg to a scratch directory, builds the reference's
own Cython kernel there (so the reference runs with its default 'compiled'
backend), imports ``swarmfilter`` from that copy and records inputs and
outputs of the hot path.  Nothing from the reference is copied into the repo
-- only the numbers it produced.  Problems for configs 2+ come from this
repo's seeded scenario generator and are stored alongside the outputs.
"""
from __future__ import annotations

import json
import os
import shutil
import subprocess
import sys
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
REF = Path("/root/reference/pkg")
SCRATCH = Path("/tmp/sgsf_golden_refbuild")


def import_reference():
    if not (SCRATCH / "src" / "swarmfilter").exists():
        shutil.rmtree(SCRATCH, ignore_errors=True)
        shutil.copytree(REF, SCRATCH)
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=SCRATCH,
                       check=True, capture_output=True)
    sys.path.insert(0, str(SCRATCH / "src"))
    import swarmfilter
    from swarmfilter import kernels
    assert kernels.active_backend() == "compiled", kernels.available_backends()
    return swarmfilter


def doc_of(problem) -> dict:
    def ep(e):
        return {"p": e.position.tolist(), "v": e.velocity.tolist(), "a": e.acceleration.tolist()}
    return {"n": problem.n, "H": problem.horizon_samples - 1, "T": problem.duration,
            "a": problem.shape.lateral, "b": problem.shape.vertical,
            "workspace": {"center": problem.workspace.center.tolist(), "a_w": problem.workspace.lateral,
                          "b_w": problem.workspace.vertical},
            "boundary": [{"start": ep(rb.start), "goal": ep(rb.goal)} for rb in problem.boundary]}


def solve_case(sfm, name, problem, proposals, degree=10, inits=None, with_svars=False, **cfg):
    config = sfm.SolverConfig(**cfg)
    filt = sfm.SafetyFilter(problem, degree=degree, config=config)
    batch = filt.batch_solve(list(proposals), inits=inits)
    B = len(batch.results)
    dim = filt.coeff_dim
    maxit = config.max_iters
    out = {
        "proposals": np.asarray(proposals, dtype=float),
        "coeffs": np.full((B, dim), np.nan), "multipliers": np.full((B, dim), np.nan),
        "res_inf": np.full((B, maxit), np.nan), "res_l2": np.full((B, maxit), np.nan),
        "iterations": np.zeros(B, np.int32), "converged": np.zeros(B, bool),
        "displacement": np.full(B, np.nan), "feasible": np.zeros(B, bool),
        "pair_margin_min": np.full(B, np.nan), "ws_margin_max": np.full(B, np.nan),
        "pair_viol": np.zeros(B, np.int32), "ws_viol": np.zeros(B, np.int32),
    }
    if inits is not None:
        out["xi0"] = np.asarray([i[0] for i in inits], dtype=float)
        out["lam0"] = np.asarray([i[1] for i in inits], dtype=float)
    errors = []
    feas_idx = {i for i, _ in sfm.metrics.feasible_results(batch.results, problem)}
    for s, r in enumerate(batch.results):
        errors.append(r.error)
        if r.coeffs is None:
            continue
        out["coeffs"][s] = r.coeffs
        out["multipliers"][s] = r.multipliers
        out["res_inf"][s, :r.iterations] = r.residual_inf
        out["res_l2"][s, :r.iterations] = r.residual_l2
        out["iterations"][s] = r.iterations
        out["converged"][s] = r.converged
        out["displacement"][s] = r.displacement
        out["feasible"][s] = s in feas_idx
        traj = sfm.coeffs_to_trajectory(r.coeffs, filt.basis, problem.n)
        rep = sfm.check_original_constraints(traj, problem, tol=1e-3)
        out["pair_margin_min"][s] = rep.pair_margin_min
        out["ws_margin_max"][s] = rep.workspace_margin_max
        out["pair_viol"][s] = rep.pair_violation_count
        out["ws_viol"][s] = rep.workspace_violation_count
        if with_svars and r.svars is not None:
            for key in ("pair_azimuth", "pair_polar", "pair_radial", "ws_azimuth", "ws_polar", "ws_radial"):
                out.setdefault("svars_" + key, []).append(getattr(r.svars, key))
    for key in list(out):
        if key.startswith("svars_"):
            out[key] = np.asarray(out[key])
    meta = {"name": name, "problem": doc_of(problem), "degree": degree,
            "config": {"rho": config.rho, "max_iters": config.max_iters, "tol_residual": config.tol_residual,
                       "tol_eq": config.tol_eq, "early_stop": config.early_stop},
            "errors": errors, "reference_backend": "compiled"}
    np.savez_compressed(HERE / f"{name}.npz", meta=np.array(json.dumps(meta)), **out)
    its = out["iterations"].tolist()
    print(f"{name}: B={B} iterations={its if B <= 12 else (min(its), max(its))} "
          f"feasible={int(out['feasible'].sum())}/{B}")


def make_problem(sfm, starts, goals, a=0.6, b=0.4, a_w=5.0, b_w=5.0, center=(0.0, 0.0, 0.0),
                 horizon_samples=51, duration=5.0):
    """Same defaults as the reference tests' conftest.make_problem."""
    bnd = tuple(sfm.RobotBoundary(start=sfm.EndpointState(position=s), goal=sfm.EndpointState(position=g))
                for s, g in zip(starts, goals))
    return sfm.SwarmProblem(n=len(bnd), horizon_samples=horizon_samples, duration=duration,
                            shape=sfm.RobotShape(lateral=a, vertical=b),
                            workspace=sfm.Workspace(center=np.asarray(center, float), lateral=a_w, vertical=b_w),
                            boundary=bnd)


def main():
    sfm = import_reference()
    from swarmfilter.proposals import straight_line_coeffs
    sys.path.insert(0, str(REPO))
    from paper_2501_19042_b200.scenarios import random_swarm_doc

    # config 1: crossing4, 8 sampled proposals (seed 0), SF 100 iterations
    c4 = sfm.load_problem(REF / "scenarios" / "crossing4.json")
    basis = sfm.build_basis(c4.duration, degree=10, samples=c4.horizon_samples)
    props = sfm.sample_proposals(c4, basis, 8, seed=0).proposals
    solve_case(sfm, "crossing4_cfg1", c4, props, max_iters=100, with_svars=True)
    # `swarmfilter generate crossing4` defaults: 50 proposals seed 0, <= 200 iterations
    props50 = sfm.sample_proposals(c4, basis, 50, seed=0).proposals
    solve_case(sfm, "crossing4_gen50", c4, props50)
    # crossing4 with early stop disabled (fixed 100 iterations)
    solve_case(sfm, "crossing4_fixed", c4, props[:3], max_iters=60, early_stop=False)
    # asymmetric 2-robot scenario of test_kernels.py:192-195 (34 iterations)
    asym = make_problem(sfm, [(1.5, 0.3, 1.0), (-1.5, -0.2, 0.9)], [(-1.5, 0.1, 1.1), (1.5, -0.3, 1.0)])
    b51 = sfm.build_basis(5.0, degree=10, samples=51)
    xa = straight_line_coeffs(asym, b51)
    solve_case(sfm, "asym2", asym, [xa], with_svars=True)
    # warm start from the asym2 result (must finish in fewer iterations)
    prior = sfm.SafetyFilter(asym, degree=10).solve(xa)
    solve_case(sfm, "asym2_warm", asym, [xa], inits=[(prior.coeffs, prior.multipliers)])
    # antipodal swap (test_solver.py:218-232; ulp-chaotic, frozen at 101)
    anti = make_problem(sfm, [(2.0, 0.0, 1.0), (-2.0, 0.0, 1.0)], [(-2.0, 0.0, 1.0), (2.0, 0.0, 1.0)])
    xs = straight_line_coeffs(anti, b51)
    solve_case(sfm, "antipodal2", anti, [xs])
    for k in (1, 2, 5, 17):
        solve_case(sfm, f"antipodal2_it{k}", anti, [xs], max_iters=k)
    # parallel lanes: feasible straight line converges in one iteration (test_solver.py:209-216)
    par = make_problem(sfm, [(0.0, 1.0, 0.0), (0.0, -1.0, 0.0)], [(1.0, 1.0, 0.0), (1.0, -1.0, 0.0)])
    eqp = sfm.build_equality(par, b51)
    xp = sfm.project_to_boundary(straight_line_coeffs(par, b51), eqp)
    solve_case(sfm, "parallel2", par, [xp])
    # single robot (no pair block)
    one = make_problem(sfm, [(1.0, 0.5, 0.0)], [(-1.0, -0.5, 0.0)], a_w=2.0, b_w=1.5)
    eq1 = sfm.build_equality(one, b51)
    base1 = straight_line_coeffs(one, b51).reshape(3, 1, 11)
    p1 = []
    for bump in ((0.0, 0.0, 3.0), (2.5, -1.0, 0.5), (-1.5, 2.0, -2.0)):
        c = base1.copy()
        c[:, 0, 3:8] += np.asarray(bump)[:, None]
        p1.append(sfm.project_to_boundary(c.ravel(), eq1))
    solve_case(sfm, "single1", one, p1)
    # degree 7, n=3 (non-default degree)
    tri = make_problem(sfm, [(2.0, 0.0, 0.0), (-1.0, 1.5, 0.5), (-1.0, -1.5, -0.5)],
                       [(-2.0, 0.0, 0.0), (1.0, -1.5, -0.5), (1.0, 1.5, 0.5)], horizon_samples=31, duration=3.0)
    b31 = sfm.build_basis(3.0, degree=7, samples=31)
    pt = sfm.sample_proposals(tri, b31, 4, seed=9).proposals
    solve_case(sfm, "tri_deg7", tri, pt, degree=7, max_iters=300)
    # n=8, H=60 seeded scenario
    p8 = sfm.load_problem(random_swarm_doc(8, 60, seed=14))
    b8 = sfm.build_basis(p8.duration, degree=10, samples=p8.horizon_samples)
    solve_case(sfm, "swarm8", p8, sfm.sample_proposals(p8, b8, 6, seed=1, spread=0.5).proposals, max_iters=400)
    # config 2 scenario: n=16, H=100 (seed 2), 4 proposals, 500 iterations
    p16 = sfm.load_problem(random_swarm_doc(16, 100, seed=2))
    b16 = sfm.build_basis(p16.duration, degree=10, samples=p16.horizon_samples)
    solve_case(sfm, "swarm16_cfg2", p16, sfm.sample_proposals(p16, b16, 4, seed=0).proposals, max_iters=500)

    # spherical-projection kernel vectors (test_kernels.py:27-34 style inputs incl. degenerate rows)
    rng = np.random.default_rng(20)
    d = rng.standard_normal((3, 400)) * 2.0
    d[:, 0] = 0.0
    d[:, 1] = (0.0, 0.0, 1.3)
    d[:, 2] = (1e-300, 0.0, 0.0)
    d[:, 3] = (0.4, 0.0, 0.0)
    d[:, 4] = (0.0, 0.7, 0.0)
    d[:, 5] = (-0.5, 0.0, 0.0)
    d[:, 6] = (0.0, 0.0, -0.9)
    d[:, 7] = (0.3, -0.2, 0.0)
    d[:, 8] = (0.0, -0.2, 0.5)
    d[:, 9] = (-0.3, 0.0, 0.25)
    d[:, 10:60] *= 0.05
    kat = {"d": d}
    from swarmfilter.kernels import spherical_project
    for tag, (lat, vert, lo, hi) in {"pair": (0.6, 0.4, 1.0, np.inf), "ws": (5.0, 3.0, 0.0, 1.0),
                                     "unit_pair": (1.0, 1.0, 1.0, np.inf), "unit_ws": (1.0, 1.0, 0.0, 1.0)}.items():
        outs = spherical_project(d[0].copy(), d[1].copy(), d[2].copy(), lat, vert, lo, hi)
        kat[tag] = np.stack([np.asarray(o) for o in outs])
        kat[tag + "_params"] = np.array([lat, vert, lo, hi])
    np.savez_compressed(HERE / "spherical_kat.npz", **kat)
    print("spherical_kat: 400 terms x 4 parameter sets")

    # step functions on the reference tests' small_setup (n=3, degree 5, 7 samples)
    small = make_problem(sfm, [(2.0, 0.0, 0.0), (-1.0, 1.5, 0.5), (-1.0, -1.5, -0.5)],
                         [(-2.0, 0.0, 0.0), (1.0, -1.5, -0.5), (1.0, 1.5, 0.5)], horizon_samples=7, duration=2.0)
    bs = sfm.build_basis(2.0, degree=5, samples=7)
    eqs = sfm.build_equality(small, bs)
    ops = sfm.build_pairwise_operator(small, bs)
    steps = {"problem": np.array(json.dumps(doc_of(small)))}
    rows = []
    for seed in range(6):
        r = np.random.default_rng(100 + seed)
        xi = r.standard_normal(ops.coeff_dim)
        lam = r.standard_normal(ops.coeff_dim)
        e = r.standard_normal(ops.rows)
        rho = float(r.uniform(0.2, 2.0))
        mu = sfm.multiplier_update(lam, xi, e, ops, rho)
        cs = sfm.coefficient_step(xi, e, lam, eqs, ops, rho)
        pb = sfm.project_to_boundary(xi, eqs)
        rows.append((xi, lam, e, rho, mu, cs, pb))
    for k, key in enumerate(("xi", "lam", "e", "rho", "mult_update", "coef_step", "projected")):
        steps[key] = np.asarray([row[k] for row in rows])
    np.savez_compressed(HERE / "steps_small.npz", **steps)
    print("steps_small: 6 random multiplier/coefficient/projection cases")


if __name__ == "__main__":
    main()
