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


def test_multi_scenario_training_runs():
    """train_init_net_multi: mixed-context batches through several problems' unrolled SFs."""
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, sample_proposals
    from paper_2501_19042_b200.initnet import InitNet, train_init_net_multi
    from paper_2501_19042_b200.scenarios import random_swarm
    torch.manual_seed(0)
    scen = []
    for s in range(3):
        sf = SafetyFilter(random_swarm(8, 20, seed=10 + s), config=SolverConfig())
        scen.append((sf, torch.from_numpy(sample_proposals(sf.problem, sf.basis, 128, seed=1).proposals).cuda()))
    net = InitNet(8, scen[0][0].coeff_dim)
    log = train_init_net_multi(scen, net, iters=3, steps=12, batch=96, per_step=3)
    assert log.steps == 12 and np.isfinite(log.losses).all() and log.sf_seconds > 0


def test_folded_init_net_equals_the_module():
    """FoldedInitNet (context encoder folded into the first layer's bias, batch norms into the Linears)
    returns the eval-mode module's (xi_0, lambda_0) to FP32 rounding."""
    import torch

    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, sample_proposals
    from paper_2501_19042_b200.initnet import FoldedInitNet, InitNet
    from paper_2501_19042_b200.scenarios import config_problem
    from paper_2501_19042_b200.unrolled import device_constants_of
    prob = config_problem(2)
    sf = SafetyFilter(prob, config=SolverConfig(max_iters=20, svars=False))
    torch.manual_seed(0)
    net = InitNet(prob.n, sf.coeff_dim).cuda()
    with torch.no_grad():   # non-trivial batch norm statistics and last layer
        for m in net.modules():
            if isinstance(m, torch.nn.BatchNorm1d):
                m.running_mean.uniform_(-0.5, 0.5)
                m.running_var.uniform_(0.5, 2.0)
        net.mlp[-1].weight.normal_(0.0, 1e-3)
    net.eval()
    xb = torch.from_numpy(sample_proposals(prob, sf.basis, 64, seed=1).proposals).cuda()
    ctx = device_constants_of(sf, "cuda")["context"][None]
    torch.backends.cuda.matmul.allow_tf32 = False
    with torch.no_grad(), torch.backends.cudnn.flags(enabled=True, allow_tf32=False):
        x_ref, l_ref = net(ctx.expand(64, -1, -1), xb)
    x_f, l_f = FoldedInitNet(net, ctx)(xb)
    assert float((x_f - x_ref).abs().max()) <= 1e-5 * float(x_ref.abs().max())
    assert float((l_f - l_ref).abs().max()) <= 1e-4 * max(float(l_ref.abs().max()), 1e-6) + 1e-7
