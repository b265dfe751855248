"""Config 5 on the GPU: training the init network through the differentiable SF kernels lowers the
paper's loss, and the initialisation sweep reports every strategy."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_training_lowers_the_loss_and_sweep_runs():
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, sample_proposals
    from paper_2501_19042_b200.initnet import STRATEGIES, InitNet, init_sweep, train_init_net
    from paper_2501_19042_b200.problem import load_problem
    from paper_2501_19042_b200.scenarios import random_swarm_doc
    torch.manual_seed(0)
    prob = load_problem(random_swarm_doc(8, 20, 3))
    sf = SafetyFilter(prob, config=SolverConfig(max_iters=300))
    pool = torch.from_numpy(sample_proposals(prob, sf.basis, 512, seed=1, spread=0.5).proposals).cuda()
    net = InitNet(prob.n, sf.coeff_dim)
    log = train_init_net(sf, net, pool, iters=5, steps=60, batch=128, lr=1e-3)
    assert log.steps == 60 and log.sf_seconds > 0
    first, last = np.mean(log.losses[:5]), np.mean(log.losses[-5:])
    assert np.isfinite(log.losses).all() and last < first
    evalset = torch.from_numpy(sample_proposals(prob, sf.basis, 64, seed=2, spread=0.5).proposals).cuda()
    res = init_sweep(sf, evalset, net, max_iters=300, trace_iters=20)
    assert set(res) == set(STRATEGIES)
    for s, r in res.items():
        assert 1 <= r["mean_iterations"] <= 300 and 0 <= r["converged"] <= 1
        assert len(r["residual_trace"]) == 20
