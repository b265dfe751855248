"""Init network (config 5) host-side checks: context features, shapes, the zero-initialised head
(an untrained net starts the SF from the raw proposal), robot-permutation invariance of the context
encoder."""
import numpy as np
import torch

from paper_2501_19042_b200.initnet import InitNet, context_features
from paper_2501_19042_b200.scenarios import config_problem


def test_context_features_layout():
    prob = config_problem(1)
    ctx = context_features(prob)
    assert ctx.shape == (18, prob.n)
    rb = prob.boundary[2]
    np.testing.assert_array_equal(ctx[0:3, 2], rb.start.position)
    np.testing.assert_array_equal(ctx[9:12, 2], rb.goal.position)


def test_untrained_net_returns_the_proposal():
    prob = config_problem(1)
    dim = 3 * prob.n * 11
    net = InitNet(prob.n, dim).eval()
    ctx = torch.as_tensor(context_features(prob)).expand(5, -1, -1)
    xb = torch.randn(5, dim, dtype=torch.float64)
    xi0, lam0 = net(ctx, xb)
    assert xi0.dtype == torch.float64 and xi0.shape == (5, dim) and lam0.shape == (5, dim)
    assert torch.equal(xi0, xb) and torch.count_nonzero(lam0) == 0


def test_context_encoder_is_permutation_invariant():
    prob = config_problem(1)
    net = InitNet(prob.n, 3 * prob.n * 11).eval()
    ctx = torch.as_tensor(context_features(prob)).unsqueeze(0).float()
    perm = torch.tensor([2, 0, 3, 1])
    a = net.point(ctx).amax(dim=2)
    b = net.point(ctx[:, :, perm]).amax(dim=2)
    assert torch.allclose(a, b, rtol=0, atol=1e-6)
