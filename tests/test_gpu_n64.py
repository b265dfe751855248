"""64-robot swarms (BASELINE config 4 size) on the GPU: the K1L kernel (sf_large.cuh).

Parity with the oracle at a fixed iteration count (both sides run the same
number of steps, no early stop), in both precisions; config 4 itself is
checked through the oracle-free properties.
"""
import numpy as np
import pytest
import torch

from oracle import sf_oracle

pytestmark = pytest.mark.gpu


def _setup(n, horizon, seed, count, max_iters, precision):
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, sample_proposals
    from paper_2501_19042_b200.problem import load_problem
    from paper_2501_19042_b200.scenarios import random_swarm_doc
    doc = random_swarm_doc(n, horizon, seed)
    prob = load_problem(doc)
    cfg = SolverConfig(max_iters=max_iters, early_stop=False, svars=False, precision=precision)
    sf = SafetyFilter(prob, config=cfg)
    props = sample_proposals(prob, sf.basis, count, seed=seed).proposals
    return doc, sf, cfg, props


@pytest.mark.parametrize("precision,n,rtol", [("lean", 64, 1e-5), ("strict", 64, 1e-9), ("lean", 40, 1e-5)])
def test_large_n_matches_oracle_fixed_iterations(precision, n, rtol):
    doc, sf, cfg, props = _setup(n, 20, 4, 2, 12, precision)
    out = sf.solve_batched(torch.from_numpy(props).cuda(), config=cfg)
    op = sf_oracle.make_problem(doc, degree=10)
    coeffs = out.coeffs.cpu().numpy()
    rinf = out.residual_inf.cpu().numpy()
    lam = out.multipliers.cpu().numpy()
    for b, x in enumerate(props):
        r = sf_oracle.solve(op, x, max_iters=12, early_stop=False)
        scale = np.abs(r.coeffs).max()
        assert np.abs(coeffs[b] - r.coeffs).max() <= rtol * scale, b
        lscale = max(np.abs(r.multipliers).max(), 1e-12)
        assert np.abs(lam[b] - r.multipliers).max() <= (1e-4 if precision == "lean" else 1e-8) * lscale, b
        np.testing.assert_allclose(rinf[b], r.residual_inf, rtol=1e-3 if precision == "lean" else 1e-7, atol=1e-9)
    assert (out.iterations.cpu().numpy() == 12).all()
    assert out.eq_err.max().item() <= 1e-8


def test_config4_properties():
    """BASELINE config 4 (64 drones, H=150): endpoint conditions to 1e-8, histories consistent with
    `converged`, verdict within converged, launch-shape invariance (a 592-sample slice of the batch)."""
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, sample_proposals
    from paper_2501_19042_b200.scenarios import config_problem
    prob = config_problem(4)
    cfg = SolverConfig(max_iters=200, svars=False)
    sf = SafetyFilter(prob, config=cfg)
    B = 592
    xb = torch.from_numpy(sample_proposals(prob, sf.basis, B, seed=0).proposals).cuda()
    out = sf.solve_batched(xb, config=cfg)
    its = out.iterations.cpu().numpy()
    conv = out.converged.cpu().numpy().astype(bool)
    feas = out.feasible.cpu().numpy().astype(bool)
    rinf = out.residual_inf.cpu().numpy()
    assert (out.status.cpu().numpy() == 0).all()
    assert out.eq_err.max().item() <= 1e-8
    assert np.all(feas <= conv)
    last = rinf[np.arange(B), its - 1]
    assert np.all((last <= 1e-3) == conv)
    alt = sf.solve_batched(xb[:64], config=cfg, grid=7)
    assert torch.equal(alt.coeffs, out.coeffs[:64]) and torch.equal(alt.iterations, out.iterations[:64])


def test_large_n_long_run_matches_oracle():
    """60 iterations at 40 robots: long enough for K1L's quiet steps (near list + motion bound) to carry
    most of the pass, against the oracle's plain every-term evaluation."""
    doc, sf, cfg, props = _setup(40, 30, 9, 2, 60, "lean")
    out = sf.solve_batched(torch.from_numpy(props).cuda(), config=cfg)
    op = sf_oracle.make_problem(doc, degree=10)
    coeffs = out.coeffs.cpu().numpy()
    rinf = out.residual_inf.cpu().numpy()
    rl2 = out.residual_l2.cpu().numpy()
    for b, x in enumerate(props):
        r = sf_oracle.solve(op, x, max_iters=60, early_stop=False)
        assert np.abs(coeffs[b] - r.coeffs).max() <= 1e-5 * np.abs(r.coeffs).max(), b
        np.testing.assert_allclose(rinf[b], r.residual_inf, rtol=1e-3, atol=1e-9)
        np.testing.assert_allclose(rl2[b], r.residual_l2, rtol=1e-3, atol=1e-9)


@pytest.mark.parametrize("precision", ["strict", "hybrid"])
def test_k1l_long_horizon_layout_fallback(precision):
    """64 robots at H = 170: in FP64 phase B's partials do not fit next to the state, so the launcher lays
    out the one-warp exact pass (SolveParams.large_coop = 0); both layouts solve."""
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, load_problem, sample_proposals
    from paper_2501_19042_b200.scenarios import random_swarm_doc
    prob = load_problem(random_swarm_doc(64, 170, 5))
    cfg = SolverConfig(max_iters=10, svars=False, precision=precision)
    sf = SafetyFilter(prob, degree=10, config=cfg)
    x = torch.from_numpy(sample_proposals(prob, sf.basis, 2, seed=1).proposals).cuda()
    out = sf.solve_batched(x, config=cfg)
    assert (out.status == 0).all() and out.eq_err.max().item() <= 1e-8
