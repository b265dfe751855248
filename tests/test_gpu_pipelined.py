"""SafetyFilter.solve_pipelined (batches on alternating side streams, two in flight) returns exactly what
solve_batched returns for each batch, with host copies in / out on the batch's own stream."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_pipelined_batches_equal_sequential_ones():
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, sample_proposals
    from paper_2501_19042_b200.scenarios import config_problem
    prob = config_problem(2)
    cfg = SolverConfig(max_iters=120, svars=False)
    sf = SafetyFilter(prob, degree=10, config=cfg)
    xs = [torch.from_numpy(sample_proposals(prob, sf.basis, b, seed=s).proposals).cuda()
          for b, s in ((300, 0), (17, 1), (450, 2), (1, 3))]
    seq = [sf.solve_batched(x, config=cfg) for x in xs]
    pipe = sf.solve_pipelined(iter(xs), config=cfg)
    torch.cuda.synchronize()
    assert len(pipe) == len(seq)
    for a, b in zip(seq, pipe):
        for k in ("coeffs", "multipliers", "iterations", "feasible", "status", "eq_err"):
            assert torch.equal(getattr(a, k), getattr(b, k)), k
        ha, hb = a.residual_inf.cpu(), b.residual_inf.cpu()   # valid up to each sample's iteration count
        for s, it in enumerate(a.iterations.tolist()):
            assert torch.equal(ha[s, :it], hb[s, :it]), s


def test_pipelined_host_copies():
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, sample_proposals
    from paper_2501_19042_b200.scenarios import config_problem
    prob = config_problem(2)
    cfg = SolverConfig(max_iters=80, svars=False)
    sf = SafetyFilter(prob, degree=10, config=cfg)
    hosts = [torch.from_numpy(sample_proposals(prob, sf.basis, 64, seed=s).proposals).pin_memory() for s in range(5)]
    got = [torch.empty(64, dtype=torch.int32).pin_memory() for _ in hosts]

    def h2d(k, x):
        return x.to("cuda", non_blocking=True)

    def d2h(k, out):
        got[k].copy_(out.iterations, non_blocking=True)

    sf.solve_pipelined(iter(hosts), config=cfg, prepare=h2d, finish=d2h)
    torch.cuda.synchronize()
    for h, g in zip(hosts, got):
        ref = sf.solve_batched(h.cuda(), config=cfg).iterations.cpu()
        assert np.array_equal(g.numpy(), ref.numpy())
