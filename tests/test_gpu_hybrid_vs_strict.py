"""Hybrid precision against strict (FP64 everywhere, which matches the reference on every frozen batch) on random
scenarios with early stop: identical iteration counts and verdicts (tools/hybrid_vs_strict.py runs the larger
sweep: 1920/1920 counts, 0 verdict flips over 30 scenarios of 3-32 robots)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,H,seed,spread", [(4, 30, 11, 1.0), (8, 50, 12, 0.6), (16, 100, 13, 0.25),
                                             (24, 50, 14, 1.0), (32, 30, 15, 0.6)])
def test_hybrid_counts_and_verdicts_equal_strict(n, H, seed, spread):
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, load_problem, sample_proposals
    from paper_2501_19042_b200.scenarios import random_swarm_doc
    prob = load_problem(random_swarm_doc(n, H, seed))
    outs = {}
    for prec in ("strict", "hybrid"):
        cfg = SolverConfig(max_iters=300, svars=False, precision=prec)
        sf = SafetyFilter(prob, degree=10, config=cfg)
        x = torch.from_numpy(sample_proposals(prob, sf.basis, 64, seed=seed, spread=spread).proposals).cuda()
        outs[prec] = sf.solve_batched(x, config=cfg)
    a, b = outs["strict"], outs["hybrid"]
    assert torch.equal(a.iterations, b.iterations)
    assert torch.equal(a.converged, b.converged) and torch.equal(a.feasible, b.feasible)
    err = (a.coeffs - b.coeffs).abs().max().item() / max(1.0, a.coeffs.abs().max().item())
    assert err <= 1e-6, err
