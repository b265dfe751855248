"""Reference-API semantics on the GPU: the reference's own solver tests
(test_solver.py:72-383) restated against this package, plus the step
functions, verdict, svars and trajectory entry points against the golden
vectors of the real reference.  All of them run the native sm_100a library.
"""
import ctypes
import json

import numpy as np
import pytest
import torch

from oracle import sf_oracle as so

from .conftest import load_golden

pytestmark = pytest.mark.gpu


def make_problem(starts, goals, a=0.6, b=0.4, a_w=5.0, b_w=5.0, center=(0.0, 0.0, 0.0), horizon_samples=51,
                 duration=5.0):
    from paper_2501_19042_b200 import EndpointState, RobotBoundary, RobotShape, SwarmProblem, Workspace
    bnd = tuple(RobotBoundary(EndpointState(np.asarray(s, float)), EndpointState(np.asarray(g, float)))
                for s, g in zip(starts, goals))
    return SwarmProblem(len(bnd), horizon_samples, duration, RobotShape(a, b),
                        Workspace(np.asarray(center, float), a_w, b_w), bnd)


@pytest.fixture(scope="module")
def parallel_filter():
    from paper_2501_19042_b200 import SafetyFilter
    return SafetyFilter(make_problem([(0.0, 1.0, 0.0), (0.0, -1.0, 0.0)], [(1.0, 1.0, 0.0), (1.0, -1.0, 0.0)]))


@pytest.fixture(scope="module")
def feasible_proposal(parallel_filter):
    from paper_2501_19042_b200 import project_to_boundary, straight_line_coeffs
    return project_to_boundary(straight_line_coeffs(parallel_filter.problem, parallel_filter.basis),
                               parallel_filter.equality)


@pytest.fixture(scope="module")
def two_robot_filter():
    from paper_2501_19042_b200 import SafetyFilter
    return SafetyFilter(make_problem([(2.0, 0.0, 1.0), (-2.0, 0.0, 1.0)], [(-2.0, 0.0, 1.0), (2.0, 0.0, 1.0)]))


@pytest.fixture(scope="module")
def swap_proposal(two_robot_filter):
    from paper_2501_19042_b200 import straight_line_coeffs
    return straight_line_coeffs(two_robot_filter.problem, two_robot_filter.basis)


@pytest.mark.parametrize("precision", ["lean", "strict", "hybrid"])
def test_feasible_proposal_converges_immediately(parallel_filter, feasible_proposal, precision):
    from paper_2501_19042_b200 import SolverConfig
    res = parallel_filter.solve(feasible_proposal, config=SolverConfig(precision=precision))
    assert res.converged and res.iterations == 1
    assert res.displacement <= 1e-6
    assert res.final_residual_inf <= 1e-9


def test_max_iters_one(two_robot_filter, swap_proposal):
    from paper_2501_19042_b200 import SolverConfig
    res = two_robot_filter.solve(swap_proposal, config=SolverConfig(max_iters=1))
    assert res.iterations == 1 and res.residual_inf.shape == (1,) and not res.converged


@pytest.mark.parametrize("iters", [1, 2, 5, 17])
def test_boundary_invariance_every_iteration(two_robot_filter, swap_proposal, iters):
    from paper_2501_19042_b200 import SolverConfig
    res = two_robot_filter.solve(swap_proposal, config=SolverConfig(max_iters=iters))
    assert res.iterations == iters
    assert np.abs(two_robot_filter.equality.residual(res.coeffs)).max() <= 1e-8


def test_fixed_point_consistency(parallel_filter, feasible_proposal):
    from paper_2501_19042_b200 import SolverConfig
    first = parallel_filter.solve(feasible_proposal)
    again = parallel_filter.solve(feasible_proposal, init=(first.coeffs, first.multipliers),
                                  config=SolverConfig(max_iters=1))
    assert np.abs(again.coeffs - first.coeffs).max() <= 1e-9
    assert np.abs(again.multipliers - first.multipliers).max() <= 1e-9


def test_early_stop_disabled_runs_full_budget(parallel_filter, feasible_proposal):
    from paper_2501_19042_b200 import SolverConfig
    res = parallel_filter.solve(feasible_proposal, config=SolverConfig(max_iters=7, early_stop=False))
    assert res.iterations == 7 and res.converged


def test_deterministic_repeat_and_identical_proposals(two_robot_filter, swap_proposal):
    r1 = two_robot_filter.solve(swap_proposal)
    r2 = two_robot_filter.solve(swap_proposal)
    np.testing.assert_array_equal(r1.coeffs, r2.coeffs)
    np.testing.assert_array_equal(r1.residual_inf, r2.residual_inf)
    batch = two_robot_filter.batch_solve([swap_proposal] * 3)
    for res in batch.results:
        np.testing.assert_array_equal(res.coeffs, r1.coeffs)
    assert two_robot_filter.batch_solve([swap_proposal]).results[0].iterations == r1.iterations


def test_warm_start_variants(two_robot_filter, swap_proposal):
    from paper_2501_19042_b200 import WarmStart
    prior = two_robot_filter.solve(swap_proposal)
    a = two_robot_filter.solve(swap_proposal, init=prior)
    b = two_robot_filter.solve(swap_proposal, init=(prior.coeffs, prior.multipliers))
    c = two_robot_filter.solve(swap_proposal, init=WarmStart(prior.coeffs, prior.multipliers))
    assert a.iterations == b.iterations == c.iterations < prior.iterations
    np.testing.assert_array_equal(a.coeffs, b.coeffs)
    np.testing.assert_array_equal(a.coeffs, c.coeffs)


def test_errors_and_isolation(two_robot_filter, swap_proposal):
    from paper_2501_19042_b200 import DimensionMismatch, SolveResult, SwarmFilterError
    failed = SolveResult(None, None, np.empty(0), np.empty(0), 0, False, np.nan, 0.0, error="boom")
    with pytest.raises(SwarmFilterError, match="failed result"):
        two_robot_filter.solve(swap_proposal, init=failed)
    with pytest.raises(DimensionMismatch, match="expected 66"):
        two_robot_filter.solve(np.zeros(10))
    with pytest.raises(DimensionMismatch):
        two_robot_filter.solve(swap_proposal, init=(np.zeros(5), np.zeros(66)))
    batch = two_robot_filter.batch_solve([swap_proposal, np.zeros(7), swap_proposal])
    assert batch.n_failed == 1 and "DimensionMismatch" in batch.results[1].error
    assert batch.results[1].coeffs is None
    assert batch.results[0].converged and batch.results[2].converged and batch.n_converged == 2
    with pytest.raises(DimensionMismatch, match="warm starts"):
        two_robot_filter.batch_solve([swap_proposal] * 2, inits=[None])


def test_module_level_wrappers(feasible_proposal, parallel_filter):
    from paper_2501_19042_b200 import batch_solve, solve
    res = solve(feasible_proposal, parallel_filter.problem)
    assert res.converged and res.iterations == 1
    assert batch_solve([feasible_proposal] * 2, parallel_filter.problem).n_converged == 2
    empty = batch_solve([], parallel_filter.problem)
    assert empty.results == [] and empty.wall_time == 0.0


def test_result_jsonable_nesting(parallel_filter, feasible_proposal):
    res = parallel_filter.solve(feasible_proposal)
    arr = np.asarray(res.to_jsonable(n=2)["coefficients"])
    assert arr.shape == (2, 3, 11)
    np.testing.assert_array_equal(arr[1, 2], res.coeffs.reshape(3, 2, 11)[2, 1])


# ------------------------------------------------------------------ step functions vs golden
def _small():
    from paper_2501_19042_b200 import SafetyFilter, load_problem
    st = load_golden("steps_small")
    prob = load_problem(json.loads(str(st["problem"])))
    return st, SafetyFilter(prob, degree=5)


def test_multiplier_update_matches_reference():
    from paper_2501_19042_b200 import multiplier_update
    st, sf = _small()
    for c in range(st["xi"].shape[0]):
        got = multiplier_update(st["lam"][c], st["xi"][c], st["e"][c], sf.operator, float(st["rho"][c]))
        np.testing.assert_allclose(got, st["mult_update"][c], atol=1e-12)
    lam = st["lam"][0]
    np.testing.assert_array_equal(multiplier_update(lam, st["xi"][0], st["e"][0], sf.operator, 0.0), lam)


def test_coefficient_step_matches_reference():
    from paper_2501_19042_b200 import coefficient_step, project_to_boundary
    st, sf = _small()
    for c in range(st["xi"].shape[0]):
        got = coefficient_step(st["xi"][c], st["e"][c], st["lam"][c], sf.equality, sf.operator, float(st["rho"][c]))
        np.testing.assert_allclose(got, st["coef_step"][c], atol=1e-9)
        assert np.abs(sf.equality.residual(got)).max() <= 1e-8
    # rho = 0 reduces to the boundary projection of xi_bar + lam (test_solver.py:148-155)
    got0 = coefficient_step(st["xi"][0], np.zeros(sf.operator.rows), st["lam"][0], sf.equality, sf.operator, 0.0)
    np.testing.assert_allclose(got0, project_to_boundary(st["xi"][0] + st["lam"][0], sf.equality), atol=1e-10)


def test_spherical_step_and_svars_match_reference():
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, load_problem
    case = load_golden("crossing4_cfg1")
    meta = case["meta"]
    prob = load_problem(meta["problem"])
    cfg = SolverConfig(precision="strict", **meta["config"])
    sf = SafetyFilter(prob, config=cfg)
    res = sf.batch_solve(list(case["proposals"][:3]), config=cfg)
    keys = ("pair_azimuth", "pair_polar", "pair_radial", "ws_azimuth", "ws_polar", "ws_radial")
    for s, r in enumerate(res.results):
        for key in keys:
            diff = getattr(r.svars, key) - case["svars_" + key][s]
            if "azimuth" in key:
                diff = np.angle(np.exp(1j * diff))
            assert np.abs(diff).max() <= 1e-6, key


# ------------------------------------------------------------------ verdict / trajectory / host entry
def test_verdict_matches_reference_counts():
    from paper_2501_19042_b200 import SafetyFilter, load_problem, verdict_batched
    for name in ("crossing4_gen50", "swarm16_cfg2", "crossing4_fixed"):
        case = load_golden(name)
        prob = load_problem(case["meta"]["problem"])
        sf = SafetyFilter(prob)
        c = torch.from_numpy(case["coeffs"]).cuda()
        conv = torch.from_numpy(case["converged"].astype(np.uint8)).cuda()
        v = {k: t.cpu().numpy() for k, t in verdict_batched(sf.operator, c, conv).items()}
        np.testing.assert_array_equal(v["feasible"].astype(bool), case["feasible"])
        np.testing.assert_array_equal(v["pair_viol"], case["pair_viol"])
        np.testing.assert_array_equal(v["ws_viol"], case["ws_viol"])
        np.testing.assert_allclose(v["pair_margin_min"], case["pair_margin_min"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(v["ws_margin_max"], case["ws_margin_max"], rtol=1e-9, atol=1e-12)


def test_trajectory_matches_oracle_basis():
    from paper_2501_19042_b200 import build_basis, coeffs_to_trajectory, load_problem
    case = load_golden("asym2")
    prob = load_problem(case["meta"]["problem"])
    basis = build_basis(prob.duration, 10, prob.horizon_samples)
    tr = coeffs_to_trajectory(case["coeffs"][0], basis, prob.n)
    W, Wd, Wdd = so.bernstein_basis(10, prob.horizon_samples, prob.duration)
    C = case["coeffs"][0].reshape(3, prob.n, 11)
    np.testing.assert_allclose(tr.positions, np.moveaxis(C @ W.T, 0, -1), atol=1e-12)
    np.testing.assert_allclose(tr.velocities, np.moveaxis(C @ Wd.T, 0, -1), atol=1e-11)
    np.testing.assert_allclose(tr.accelerations, np.moveaxis(C @ Wdd.T, 0, -1), atol=1e-10)


def test_solve_host_entry_point():
    """sgsf_solve_host: host buffers in/out through the C ABI (the ctypes binding of INTEGRATION.md)."""
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, load_problem, native
    case = load_golden("crossing4_cfg1")
    meta = case["meta"]
    prob = load_problem(meta["problem"])
    sf = SafetyFilter(prob)
    B, dim, mi = case["proposals"].shape[0], 132, meta["config"]["max_iters"]
    xb = np.ascontiguousarray(case["proposals"])
    coeffs = np.empty((B, dim))
    mult = np.empty((B, dim))
    rinf = np.empty((B, mi))
    rl2 = np.empty((B, mi))
    its = np.empty(B, np.int32)
    conv = np.empty(B, np.uint8)
    feas = np.empty(B, np.uint8)
    disp = np.empty(B)
    status = np.empty(B, np.int32)
    cfg = native.Config(mi, 1e-3, 1e-8, 1, native.PRECISION_LEAN, 0, 0, 0)
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    rc = native.load().sgsf_solve_host(sf.operator.handle(1.0), B, P(xb), None, None, None, ctypes.byref(cfg),
                                       P(coeffs), P(mult), P(rinf), P(rl2), P(its), P(conv), P(feas), P(disp),
                                       P(status), None)
    native.check(rc, "sgsf_solve_host")
    np.testing.assert_array_equal(its, case["iterations"])
    np.testing.assert_array_equal(feas.astype(bool), case["feasible"])
    assert np.abs(coeffs - case["coeffs"]).max() <= 1e-5 * np.abs(case["coeffs"]).max()


def test_full_size_config2_properties():
    """BASELINE config 2 at full size (1000 samples): properties that need no oracle --
    endpoint conditions held to 1e-8, converged samples' histories end at/below tol,
    verdicts consistent with converged, and results independent of launch shape."""
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, sample_proposals
    from paper_2501_19042_b200.scenarios import config_problem
    prob = config_problem(2)
    cfg = SolverConfig(max_iters=500, svars=False)
    sf = SafetyFilter(prob, config=cfg)
    xb = torch.from_numpy(sample_proposals(prob, sf.basis, 1000, seed=0).proposals).cuda()
    out = sf.solve_batched(xb, config=cfg)
    its = out.iterations.cpu().numpy()
    conv = out.converged.cpu().numpy().astype(bool)
    feas = out.feasible.cpu().numpy().astype(bool)
    rinf = out.residual_inf.cpu().numpy()
    assert (out.status.cpu().numpy() == 0).all()
    assert out.eq_err.max().item() <= 1e-8
    assert np.all(feas <= conv)
    last = rinf[np.arange(1000), its - 1]
    assert np.all((last <= 1e-3) == conv)
    assert conv.mean() > 0.5
    alt = sf.solve_batched(xb, config=cfg, slots_per_block=1, grid=37)
    assert torch.equal(alt.coeffs, out.coeffs) and torch.equal(alt.iterations, out.iterations)
