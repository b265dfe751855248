"""Differentiable SF on the GPU (``sgsf_unroll`` / ``sgsf_unroll_backward``) against the autograd oracle.

Forward: every iterate equals the oracle's (the reference step, FP64) to 1e-10 relative.  Backward:
dL/d(xi_bar, xi0, lambda0) of a random linear functional of all iterates, and of the paper's loss
through the default boundary-projection start, equal torch autograd through the oracle to 1e-8
relative.  Cases cover active pair and workspace terms, several window shapes (n = 8, 16, 40) and
the full config-2 horizon.
"""
import numpy as np
import pytest
import torch

from oracle import sf_oracle
from oracle import sf_unroll_oracle as uo

pytestmark = pytest.mark.gpu


def _case(n, horizon, seed, spread, count):
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, sample_proposals
    from paper_2501_19042_b200.problem import load_problem
    from paper_2501_19042_b200.scenarios import random_swarm_doc
    doc = random_swarm_doc(n, horizon, seed)
    prob = load_problem(doc)
    sf = SafetyFilter(prob, config=SolverConfig())
    props = sample_proposals(prob, sf.basis, count, seed=seed, spread=spread).proposals
    op = sf_oracle.make_problem(doc, degree=10)
    return sf, op, props


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("n,horizon,seed,spread,iters", [(8, 20, 3, 1.5, 6), (16, 100, 2, 1.0, 4), (40, 20, 1, 1.0, 3)])
def test_forward_iterates_match_oracle(n, horizon, seed, spread, iters):
    from paper_2501_19042_b200 import unrolled_solve
    sf, op, props = _case(n, horizon, seed, spread, 2)
    tp = uo.TorchProblem(op)
    rng = np.random.default_rng(seed)
    lam0 = rng.normal(0, 0.05, props.shape)
    x0 = np.stack([sf_oracle.project_boundary(op, x) for x in props])
    out = unrolled_solve(sf, torch.from_numpy(props).cuda(), torch.from_numpy(x0).cuda(),
                         torch.from_numpy(lam0).cuda(), iters=iters)
    xs = out.coeffs.cpu().numpy()
    ls = out.multipliers.cpu().numpy()
    for b in range(props.shape[0]):
        rx, rl = uo.unroll(tp, torch.tensor(props[b]), torch.tensor(x0[b]), torch.tensor(lam0[b]), iters)
        assert _rel(xs[b], rx.numpy()) <= 1e-10
        assert _rel(ls[b], rl.numpy()) <= 1e-10


@pytest.mark.parametrize("n,horizon,seed,spread,iters", [(8, 20, 3, 1.5, 5), (16, 100, 2, 1.0, 4), (40, 20, 1, 1.0, 3)])
def test_backward_matches_autograd(n, horizon, seed, spread, iters):
    from paper_2501_19042_b200 import unrolled_solve
    sf, op, props = _case(n, horizon, seed, spread, 2)
    tp = uo.TorchProblem(op)
    rng = np.random.default_rng(seed + 10)
    lam0 = rng.normal(0, 0.05, props.shape)
    x0 = np.stack([sf_oracle.project_boundary(op, x) for x in props])
    gx = rng.normal(size=(props.shape[0], iters + 1, props.shape[1]))
    gl = rng.normal(size=gx.shape)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().requires_grad_(True)
    xb_t, x0_t, l0_t = dev(props), dev(x0), dev(lam0)
    out = unrolled_solve(sf, xb_t, x0_t, l0_t, iters=iters)
    loss = (out.coeffs * torch.from_numpy(gx).cuda()).sum() + (out.multipliers * torch.from_numpy(gl).cuda()).sum()
    loss.backward()
    for b in range(props.shape[0]):
        g_xb, g_x0, g_l0, _, _ = uo.gradients(tp, props[b], x0[b], lam0[b], iters, gx[b], gl[b])
        assert _rel(xb_t.grad[b].cpu().numpy(), g_xb) <= 1e-8
        assert _rel(x0_t.grad[b].cpu().numpy(), g_x0) <= 1e-8
        assert _rel(l0_t.grad[b].cpu().numpy(), g_l0) <= 1e-8


def test_paper_loss_gradient_through_default_start():
    """fixed_point_loss (eq. NN_loss) from the default start (boundary projection, zero multipliers):
    the gradient with respect to the proposal equals autograd through the oracle."""
    from paper_2501_19042_b200 import fixed_point_loss, unrolled_solve
    sf, op, props = _case(8, 20, 3, 1.5, 3)
    tp = uo.TorchProblem(op)
    iters = 5
    xb = torch.from_numpy(props).cuda().requires_grad_(True)
    out = unrolled_solve(sf, xb, iters=iters)
    fixed_point_loss(out, xb, reduction="sum").backward()
    for b in range(props.shape[0]):
        x = torch.tensor(props[b], requires_grad=True)
        x0 = uo.boundary_projection(tp, x.reshape(tp.shape)).reshape(-1)
        xs, ls = uo.unroll(tp, x, x0, torch.zeros(op.dim, dtype=torch.float64), iters)
        uo.fixed_point_loss(xs, ls, x).backward()
        assert _rel(xb.grad[b].cpu().numpy(), x.grad.numpy()) <= 1e-8


def test_forward_equals_strict_solver_and_is_deterministic():
    """The unrolled forward and the strict K1 solve (no early stop) are the same iteration; repeated
    and re-batched runs are bitwise identical."""
    from dataclasses import replace

    from paper_2501_19042_b200 import unrolled_solve
    sf, op, props = _case(16, 100, 2, 1.0, 6)
    xb = torch.from_numpy(props).cuda()
    iters = 8
    out = unrolled_solve(sf, xb, iters=iters)
    cfg = replace(sf.config, max_iters=iters, early_stop=False, precision="strict", svars=False)
    ref = sf.solve_batched(xb, config=cfg, verdict=False)
    scale = ref.coeffs.abs().max().item()
    assert (out.coeffs[:, -1] - ref.coeffs).abs().max().item() <= 1e-10 * scale
    again = unrolled_solve(sf, xb[2:5], iters=iters)
    assert torch.equal(again.coeffs, out.coeffs[2:5]) and torch.equal(again.multipliers, out.multipliers[2:5])


def test_shape_errors():
    from paper_2501_19042_b200 import DimensionMismatch, unrolled_solve
    sf, op, props = _case(8, 20, 3, 1.5, 2)
    xb = torch.from_numpy(props).cuda()
    with pytest.raises(DimensionMismatch):
        unrolled_solve(sf, xb[:, :-1])
    with pytest.raises(DimensionMismatch):
        unrolled_solve(sf, xb, xi0=xb[:1])
    out = unrolled_solve(sf, xb, iters=0)
    assert out.coeffs.shape == (2, 1, sf.coeff_dim)
