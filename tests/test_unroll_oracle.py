"""Pins the differentiable-SF oracle (``oracle/sf_unroll_oracle.py``) on the CPU.

* Its forward iterates equal ``sf_oracle.solve`` at a fixed iteration count. ``sf_oracle`` is pinned
  to the reference's golden vectors in ``test_oracle.py``.
* Its autograd gradient equals central finite differences of that forward, along random directions,
  with active pair and workspace terms present.
* The paper's loss (eq. NN_loss) is the stated sum.
"""
import numpy as np
import pytest
import torch

from oracle import sf_oracle
from oracle import sf_unroll_oracle as uo


def _case(n=8, horizon=20, seed=3, spread=1.5):
    from paper_2501_19042_b200 import sample_proposals
    from paper_2501_19042_b200.problem import load_problem
    from paper_2501_19042_b200.scenarios import random_swarm_doc
    doc = random_swarm_doc(n, horizon, seed)
    prob = load_problem(doc)
    from paper_2501_19042_b200.basis import build_basis
    basis = build_basis(prob.duration, degree=10, samples=prob.horizon_samples)
    xb = sample_proposals(prob, basis, 1, seed=seed, spread=spread).proposals[0]
    op = sf_oracle.make_problem(doc, degree=10)
    return op, xb


def _active_counts(op, C):
    pos = sf_oracle.positions(op, C.reshape(3, op.n, op.m1))
    d = sf_oracle.pair_diffs(op, pos)
    rp = np.sqrt((d[0] ** 2 + d[1] ** 2) / op.lat ** 2 + d[2] ** 2 / op.vert ** 2)
    rel = pos - op.center[:, None, None]
    rw = np.sqrt((rel[0] ** 2 + rel[1] ** 2) / op.ws_lat ** 2 + rel[2] ** 2 / op.ws_vert ** 2)
    return int((rp < 1).sum()), int((rw > 1).sum())


def test_forward_matches_pinned_oracle():
    op, xb = _case()
    tp = uo.TorchProblem(op)
    x0 = sf_oracle.project_boundary(op, xb)
    K = 6
    xs, ls = uo.unroll(tp, torch.tensor(xb), torch.tensor(x0), torch.zeros(op.dim), K)
    for k in (1, 3, K):
        r = sf_oracle.solve(op, xb, max_iters=k, early_stop=False)
        scale = np.abs(r.coeffs).max()
        assert np.abs(xs[k].numpy() - r.coeffs).max() <= 1e-11 * scale
        assert np.abs(ls[k].numpy() - r.multipliers).max() <= 1e-11 * max(np.abs(r.multipliers).max(), 1.0)
    np.testing.assert_allclose(uo.boundary_projection(tp, torch.tensor(xb).reshape(3, op.n, op.m1)).numpy().ravel(),
                               x0, rtol=0, atol=1e-12)


def test_gradient_matches_finite_differences():
    op, xb = _case()
    tp = uo.TorchProblem(op)
    x0 = sf_oracle.project_boundary(op, xb)
    l0 = np.random.default_rng(0).normal(0, 0.05, op.dim)
    K = 4
    npair, nws = _active_counts(op, x0)
    assert npair > 0 and nws > 0, "the case must exercise active pair and workspace terms"
    rng = np.random.default_rng(1)
    gx = rng.normal(size=(K + 1, op.dim))
    gl = rng.normal(size=(K + 1, op.dim))
    g_xb, g_x0, g_l0, _, _ = uo.gradients(tp, xb, x0, l0, K, gx, gl)

    def loss(a, b, c):
        xs, ls = uo.unroll(tp, torch.tensor(a), torch.tensor(b), torch.tensor(c), K)
        return float((xs.numpy() * gx).sum() + (ls.numpy() * gl).sum())

    h = 1e-6
    for which, g in ((0, g_xb), (1, g_x0), (2, g_l0)):
        v = rng.normal(size=op.dim)
        args_p = [xb.copy(), x0.copy(), l0.copy()]
        args_m = [xb.copy(), x0.copy(), l0.copy()]
        args_p[which] += h * v
        args_m[which] -= h * v
        fd = (loss(*args_p) - loss(*args_m)) / (2 * h)
        assert abs(fd - g @ v) <= 1e-5 * max(abs(fd), 1.0), (which, fd, g @ v)


def test_fixed_point_loss_definition():
    xs = torch.arange(12, dtype=torch.float64).reshape(3, 4)
    ls = torch.ones(3, 4, dtype=torch.float64)
    xb = torch.zeros(4, dtype=torch.float64)
    # steps of 4 in each of 4 coordinates, two steps: 2 * 4 * 16; lambda constant; ||xs[-1]||^2
    assert float(uo.fixed_point_loss(xs, ls, xb)) == pytest.approx(2 * 4 * 16 + float((xs[-1] ** 2).sum()))
