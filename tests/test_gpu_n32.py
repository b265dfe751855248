"""32-robot swarms (BASELINE config 3 size) on the GPU.

The 32-robot kernel variant gives each time step two lanes of 16 robots
(TPS = 2) and runs one slot per CTA.  Parity with the oracle is checked at a
fixed iteration count (no early stop), so both sides run the same number of
alternating-minimisation steps; the full config-3 batch is checked through
the oracle-free properties used for config 2.
"""
import dataclasses

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


def _oracle(doc, props, max_iters):
    op = sf_oracle.make_problem(doc, degree=10)
    return [sf_oracle.solve(op, x, max_iters=max_iters, early_stop=False) for x in props]


@pytest.mark.parametrize("precision,horizon,rtol", [("lean", 100, 1e-5), ("strict", 40, 1e-9), ("hybrid", 100, 1e-7)])
def test_n32_matches_oracle_fixed_iterations(precision, horizon, rtol):
    doc, sf, cfg, props = _setup(32, horizon, 3, 3, 25, precision)
    out = sf.solve_batched(torch.from_numpy(props).cuda(), config=cfg)
    ref = _oracle(doc, props, 25)
    coeffs = out.coeffs.cpu().numpy()
    rinf = out.residual_inf.cpu().numpy()
    for b, r in enumerate(ref):
        scale = np.abs(r.coeffs).max()
        assert np.abs(coeffs[b] - r.coeffs).max() <= rtol * scale, b
        np.testing.assert_allclose(rinf[b], r.residual_inf, rtol=1e-7 if precision == "strict" else 1e-3, atol=1e-9)
    assert (out.iterations.cpu().numpy() == 25).all()
    assert out.eq_err.max().item() <= 1e-8


def test_n32_strict_full_horizon_runs_on_k1l():
    """Strict (FP64 positions) at 32 robots and H = 100 does not fit one K1 slot; the launcher hands it to K1L
    (one CTA of eight warps per sample), which matches the oracle at fixed iterations."""
    doc, sf, cfg, props = _setup(32, 100, 3, 2, 12, "strict")
    out = sf.solve_batched(torch.from_numpy(props).cuda(), config=cfg)
    ref = _oracle(doc, props, 12)
    coeffs = out.coeffs.cpu().numpy()
    rinf = out.residual_inf.cpu().numpy()
    for b, r in enumerate(ref):
        assert np.abs(coeffs[b] - r.coeffs).max() <= 1e-9 * np.abs(r.coeffs).max(), b
        np.testing.assert_allclose(rinf[b], r.residual_inf, rtol=1e-7, atol=1e-9)
    assert out.eq_err.max().item() <= 1e-8


def test_full_size_config3_properties():
    """BASELINE config 3 (32 drones, H=100) at its full batch of 4096: endpoint conditions to 1e-8,
    histories consistent with `converged`, verdict within converged, launch-shape invariance."""
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, sample_proposals
    from paper_2501_19042_b200.scenarios import config_problem
    prob = config_problem(3)
    cfg = SolverConfig(max_iters=500, svars=False)
    sf = SafetyFilter(prob, config=cfg)
    B = 4096
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
    sub = dataclasses.replace(cfg)
    alt = sf.solve_batched(xb[:300], config=sub, grid=37)
    assert torch.equal(alt.coeffs, out.coeffs[:300]) and torch.equal(alt.iterations, out.iterations[:300])


@pytest.mark.parametrize("precision,n,horizon,degree", [("hybrid", 24, 150, 10), ("lean", 20, 160, 10),
                                                        ("hybrid", 32, 127, 15), ("strict", 16, 260, 10),
                                                        ("hybrid", 8, 420, 10)])
def test_n32_past_one_slot_runs_on_k1l(precision, n, horizon, degree):
    """Shapes where one K1 slot does not fit -- 17..32 robots past 128 time steps or with hybrid's scratch at
    H = 127 and degree 15; FP64 16 robots at H = 260; 8 robots past 384 time steps: the launcher hands the
    batch to K1L, which matches the oracle at fixed iterations."""
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, sample_proposals
    from paper_2501_19042_b200.problem import load_problem
    from paper_2501_19042_b200.scenarios import random_swarm_doc
    doc = random_swarm_doc(n, horizon, 5)
    prob = load_problem(doc)
    cfg = SolverConfig(max_iters=10, early_stop=False, svars=False, precision=precision)
    sf = SafetyFilter(prob, degree=degree, config=cfg)
    props = sample_proposals(prob, sf.basis, 2, seed=5).proposals
    out = sf.solve_batched(torch.from_numpy(props).cuda(), config=cfg)
    op = sf_oracle.make_problem(doc, degree=degree)
    rtol = 1e-5 if precision == "lean" else 1e-7
    assert (out.status == 0).all() and out.eq_err.max().item() <= 1e-8
    coeffs, rinf = out.coeffs.cpu().numpy(), out.residual_inf.cpu().numpy()
    for b, x in enumerate(props):
        r = sf_oracle.solve(op, x, max_iters=10, early_stop=False)
        assert np.abs(coeffs[b] - r.coeffs).max() <= rtol * np.abs(r.coeffs).max(), b
        np.testing.assert_allclose(rinf[b], r.residual_inf, rtol=1e-3, atol=1e-9)


@pytest.mark.parametrize("precision", ["hybrid", "lean"])
def test_n32_longest_horizon_fits_one_cta(precision):
    """32 robots at H = 127 (128 time steps, eight two-lane warps): the slot, including hybrid's
    warp-cooperative careful-path scratch, fits the 227 KB of shared memory."""
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, load_problem, sample_proposals
    from paper_2501_19042_b200.scenarios import random_swarm_doc
    prob = load_problem(random_swarm_doc(32, 127, 3))
    cfg = SolverConfig(max_iters=20, svars=False, precision=precision)
    sf = SafetyFilter(prob, degree=10, config=cfg)
    x = torch.from_numpy(sample_proposals(prob, sf.basis, 4, seed=1).proposals).cuda()
    out = sf.solve_batched(x, config=cfg)
    assert (out.status == 0).all() and out.eq_err.max().item() <= 1e-8
