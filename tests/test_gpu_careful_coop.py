"""The warp-cooperative careful path (hybrid precision, n <= 4: the FP64 reference-trig terms of the few
careful time steps -- the fixed endpoints of symmetric scenarios -- spread over the warp's lanes,
sf_persistent.cuh hy_careful_item / hy_step_coop) gives the serial path's results bit for bit."""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _solve(sf, xb, cfg, coop: bool):
    old = os.environ.get("SGSF_NO_COOP")
    os.environ["SGSF_NO_COOP"] = "0" if coop else "1"
    try:
        out = sf.solve_batched(xb, config=cfg)
        torch.cuda.synchronize()
    finally:
        if old is None:
            del os.environ["SGSF_NO_COOP"]
        else:
            os.environ["SGSF_NO_COOP"] = old
    return out


@pytest.mark.parametrize("batch,seed", [(8, 0), (64, 3)])
def test_cooperative_careful_path_is_bitwise_the_serial_one(batch, seed):
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, sample_proposals
    from paper_2501_19042_b200.scenarios import config_problem
    prob = config_problem(1)   # 4 robots crossing at one altitude: every endpoint step is careful
    cfg = SolverConfig(max_iters=100, svars=False, precision="hybrid")
    sf = SafetyFilter(prob, degree=10, config=cfg)
    xb = torch.from_numpy(sample_proposals(prob, sf.basis, batch, seed=seed).proposals).cuda()
    a, b = _solve(sf, xb, cfg, True), _solve(sf, xb, cfg, False)
    for k in ("coeffs", "iterations", "converged", "multipliers", "feasible", "status"):
        assert torch.equal(getattr(a, k), getattr(b, k)), k
    for k in ("residual_inf", "residual_l2"):   # valid up to each sample's iteration count
        ha, hb = getattr(a, k).cpu(), getattr(b, k).cpu()
        for s, it in enumerate(a.iterations.tolist()):
            assert torch.equal(ha[s, :it], hb[s, :it]), (k, s)
    assert (a.status == 0).all()


def test_cooperative_careful_path_on_the_reference_goldens():
    """crossing4_cfg1 (the real reference's output, n = 4, symmetric): identical counts, coefficients to the
    hybrid parity tolerance, with the cooperative path taken."""
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, load_problem

    from .conftest import load_golden
    case = load_golden("crossing4_cfg1")
    meta = case["meta"]
    cfg = SolverConfig(precision="hybrid", svars=False, **meta["config"])
    sf = SafetyFilter(load_problem(meta["problem"]), degree=meta["degree"], config=cfg)
    xb = torch.from_numpy(np.ascontiguousarray(case["proposals"], dtype=np.float64)).cuda()
    out = _solve(sf, xb, cfg, True)
    assert out.iterations.cpu().numpy().tolist() == case["iterations"].astype(int).tolist()
    err = np.abs(out.coeffs.cpu().numpy() - case["coeffs"]).max() / max(1.0, np.abs(case["coeffs"]).max())
    assert err <= 1e-6


def test_round_based_careful_path_n32():
    """n = 32 (config 3's last 512-sample shard has ~100 careful step-finishes): the warp-cooperative rounds
    (hy_careful_rounds) give the serial path's R rows, interior bits and stop decisions bit for bit; only the
    careful steps' l2 exit partials are summed in another order."""
    import bench
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig
    prob, shard, _ = bench.workload(3, 7, 8, None)
    cfg = SolverConfig(max_iters=500, svars=False, precision="hybrid")
    sf = SafetyFilter(prob, degree=10, config=cfg)
    xb = torch.from_numpy(shard).cuda()
    a, b = _solve(sf, xb, cfg, True), _solve(sf, xb, cfg, False)
    for k in ("coeffs", "iterations", "converged", "multipliers", "feasible", "status"):
        assert torch.equal(getattr(a, k), getattr(b, k)), k
    ha, hb = a.residual_inf.cpu(), b.residual_inf.cpu()
    la, lb = a.residual_l2.cpu(), b.residual_l2.cpu()
    for s, it in enumerate(a.iterations.tolist()):
        assert torch.equal(ha[s, :it], hb[s, :it]), s
        assert torch.allclose(la[s, :it], lb[s, :it], rtol=1e-12, atol=0), s


@pytest.mark.parametrize("precision", ["hybrid", "lean", "strict"])
def test_long_horizon_n4_fits(precision):
    """Four robots at H = 300: past 128 steps the cooperative careful path's scratch is not laid out, so the
    slot still fits one CTA (the serial careful path takes the rare careful steps)."""
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, load_problem, sample_proposals
    from paper_2501_19042_b200.scenarios import random_swarm_doc
    prob = load_problem(random_swarm_doc(4, 300, 3))
    cfg = SolverConfig(max_iters=20, svars=False, precision=precision)
    sf = SafetyFilter(prob, degree=10, config=cfg)
    x = torch.from_numpy(sample_proposals(prob, sf.basis, 4, seed=1).proposals).cuda()
    out = sf.solve_batched(x, config=cfg)
    assert (out.status == 0).all() and out.eq_err.max().item() <= 1e-8
