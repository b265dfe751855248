"""Kernel-variant coverage on the GPU, against the oracle.

* wide degree (m1 > 12 -> the 16-column variants) in every kernel family: K1 (n <= 16), K1 with two
  lanes per step (n <= 32), K1L (n <= 64);
* phantom robots inside a variant (n = 20 on the 32-robot layout, n = 48 on the 64-robot one);
* warm starts and `want_prev` on K1L (a warm start continues the iteration exactly);
* the windowed verdict and svars kernels at 40 robots.
Parity is checked at a fixed iteration count (no early stop), so both sides take the same steps.
"""
import numpy as np
import pytest
import torch

from oracle import sf_oracle

pytestmark = pytest.mark.gpu


def _setup(n, horizon, seed, count, max_iters, precision, degree=10):
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, sample_proposals
    from paper_2501_19042_b200.problem import load_problem
    from paper_2501_19042_b200.scenarios import random_swarm_doc
    doc = random_swarm_doc(n, horizon, seed)
    prob = load_problem(doc)
    cfg = SolverConfig(max_iters=max_iters, early_stop=False, svars=False, precision=precision)
    sf = SafetyFilter(prob, degree=degree, config=cfg)
    props = sample_proposals(prob, sf.basis, count, seed=seed).proposals
    return doc, sf, cfg, props


@pytest.mark.parametrize("n,degree,precision,rtol", [
    (16, 14, "lean", 1e-5), (16, 14, "strict", 1e-9),      # K1, wide
    (16, 10, "hybrid", 1e-7), (12, 14, "hybrid", 1e-7),    # K1 hybrid: tensor-core positions / FFMA, wide
    (6, 10, "hybrid", 1e-7), (28, 10, "hybrid", 1e-7),     # K1 hybrid: phantoms, two lanes per step
    (20, 10, "lean", 1e-5), (24, 13, "lean", 1e-5),        # K1 two lanes per step: phantoms, wide
    (48, 15, "lean", 1e-5), (48, 13, "strict", 1e-9),      # K1L: phantoms, wide
])
def test_variant_parity_fixed_iterations(n, degree, precision, rtol):
    horizon = 30 if n <= 24 else 20
    doc, sf, cfg, props = _setup(n, horizon, 5, 2, 10, precision, degree)
    out = sf.solve_batched(torch.from_numpy(props).cuda(), config=cfg)
    op = sf_oracle.make_problem(doc, degree=degree)
    coeffs = out.coeffs.cpu().numpy()
    lam = out.multipliers.cpu().numpy()
    rinf = out.residual_inf.cpu().numpy()
    for b, x in enumerate(props):
        r = sf_oracle.solve(op, x, max_iters=10, early_stop=False)
        assert np.abs(coeffs[b] - r.coeffs).max() <= rtol * np.abs(r.coeffs).max(), b
        lscale = max(np.abs(r.multipliers).max(), 1e-12)
        mtol = {"lean": 1e-4, "hybrid": 1e-6, "strict": 1e-8}[precision]
        assert np.abs(lam[b] - r.multipliers).max() <= mtol * lscale + 1e-12, b   # (+ the oracle's trig leaks)
        # (lean / hybrid histories are FP32-measured: differences of FP32 positions)
        np.testing.assert_allclose(rinf[b], r.residual_inf, rtol=1e-7 if precision == "strict" else 1e-3, atol=1e-9)
    assert out.eq_err.max().item() <= 1e-8


def test_large_n_warm_start_continues_the_iteration():
    """K1L: 5 iterations, then a warm start from (coeffs, multipliers) for 5 more, equals 10 straight
    iterations; `want_prev` returns the 9-iteration coefficients."""
    doc, sf, cfg, props = _setup(40, 20, 6, 3, 10, "lean")
    xb = torch.from_numpy(props).cuda()
    from dataclasses import replace
    full = sf.solve_batched(xb, config=cfg, want_prev=True)
    five = sf.solve_batched(xb, config=replace(cfg, max_iters=5))
    cont = sf.solve_batched(xb, xi0=five.coeffs, lam0=five.multipliers, config=replace(cfg, max_iters=5))
    nine = sf.solve_batched(xb, config=replace(cfg, max_iters=9))
    scale = full.coeffs.abs().max().item()
    assert (cont.coeffs - full.coeffs).abs().max().item() <= 1e-12 * scale
    assert (cont.multipliers - full.multipliers).abs().max().item() <= 1e-12 * max(full.multipliers.abs().max().item(), 1e-12)
    assert torch.equal(full.coeffs_prev, nine.coeffs)


def test_large_n_verdict_and_svars_match_oracle():
    """Windowed verdict (K2) and svars (K2b) at 40 robots, H=50: margins and counts as the oracle's
    check, spherical variables as the reference formula on the same positions."""
    from paper_2501_19042_b200.verdict import verdict_batched
    doc, sf, cfg, props = _setup(40, 50, 7, 2, 15, "lean")
    out = sf.solve_batched(torch.from_numpy(props).cuda(), config=cfg)
    op = sf_oracle.make_problem(doc, degree=10)
    v = {k: t.cpu().numpy() for k, t in verdict_batched(sf.operator, out.coeffs, None, 1e-3).items()}
    svs = sf.svars_of(out.coeffs)
    C = out.coeffs.cpu().numpy()
    for b in range(C.shape[0]):
        ref = sf_oracle.check_constraints(op, C[b], 1e-3)
        assert bool(v["ok"][b]) == ref.ok
        assert v["pair_viol"][b] == ref.pair_violation_count and v["ws_viol"][b] == ref.workspace_violation_count
        assert abs(v["pair_margin_min"][b] - ref.pair_margin_min) <= 1e-12 * max(1.0, abs(ref.pair_margin_min))
        assert abs(v["ws_margin_max"][b] - ref.workspace_margin_max) <= 1e-12 * max(1.0, abs(ref.workspace_margin_max))
        pos = sf_oracle.positions(op, C[b].reshape(3, op.n, op.m1))
        d = sf_oracle.pair_diffs(op, pos)
        pa, pp, pr, *_ = sf_oracle.spherical_project(d[0].ravel(), d[1].ravel(), d[2].ravel(), op.lat, op.vert,
                                                     1.0, np.inf)
        np.testing.assert_allclose(svs[b].pair_radial.ravel(), pr, rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(np.cos(svs[b].pair_polar.ravel()), np.cos(pp), rtol=0, atol=1e-12)


@pytest.mark.parametrize("n,degree", [(12, 10), (16, 14), (9, 13)])
def test_tensor_core_positions_variants(n, degree):
    """The 3xTF32 tcgen05 position GEMM (K1 with 97..128 steps, <= 16 robots, lean): phantom robots
    (n < 16) and the 16-column variant (degree > 11) against the oracle at a fixed iteration count."""
    doc, sf, cfg, props = _setup(n, 100, 8, 2, 10, "lean", degree)
    out = sf.solve_batched(torch.from_numpy(props).cuda(), config=cfg)
    op = sf_oracle.make_problem(doc, degree=degree)
    coeffs = out.coeffs.cpu().numpy()
    rinf = out.residual_inf.cpu().numpy()
    for b, x in enumerate(props):
        r = sf_oracle.solve(op, x, max_iters=10, early_stop=False)
        assert np.abs(coeffs[b] - r.coeffs).max() <= 1e-5 * np.abs(r.coeffs).max(), b
        np.testing.assert_allclose(rinf[b], r.residual_inf, rtol=1e-3, atol=1e-9)
    assert out.eq_err.max().item() <= 1e-8


def test_tensor_core_and_ffma_positions_agree():
    """Config 2 with the tcgen05 positions (default) and with SGSF_NO_TC=1 (packed FFMA): the same
    iterations and verdicts up to borderline flips, coefficients within the lean tolerance."""
    import os
    import subprocess
    import sys
    code = (
        "import torch, numpy as np, sys\n"
        "sys.path.insert(0, '.')\n"
        "import bench\n"
        "from paper_2501_19042_b200 import SafetyFilter\n"
        "prob, shard, cfg = bench.config2_case(300)\n"
        "sf = SafetyFilter(prob, degree=10, config=cfg)\n"
        "out = sf.solve_batched(torch.from_numpy(shard).cuda(), config=cfg)\n"
        "np.savez(sys.argv[1], c=out.coeffs.cpu().numpy(), it=out.iterations.cpu().numpy(), "
        "f=out.feasible.cpu().numpy())\n")
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        res = {}
        for tag, env in (("tc", {}), ("ffma", {"SGSF_NO_TC": "1"})):
            path = os.path.join(d, tag + ".npz")
            subprocess.run([sys.executable, "-c", code, path], check=True, env={**os.environ, **env},
                           cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
            res[tag] = np.load(path)
    it_tc, it_f = res["tc"]["it"], res["ffma"]["it"]
    same = it_tc == it_f
    assert same.mean() >= 0.95
    c_tc, c_f = res["tc"]["c"][same], res["ffma"]["c"][same]
    assert np.abs(c_tc - c_f).max() <= 1e-5 * np.abs(c_f).max()
    assert (res["tc"]["f"] == res["ffma"]["f"]).mean() >= 0.97


@pytest.mark.parametrize("horizon,count", [(96, 3), (127, 2), (100, 1)])
def test_tensor_core_positions_horizon_edges(horizon, count):
    """The tcgen05 position path at the ends of its range: S = 97 (one valid step in the last 8-step
    chunk), S = 128 (every TMEM lane a real step), and a batch of one sample."""
    doc, sf, cfg, props = _setup(16, horizon, 9, count, 8, "lean", 10)
    out = sf.solve_batched(torch.from_numpy(props).cuda(), config=cfg)
    op = sf_oracle.make_problem(doc, degree=10)
    coeffs = out.coeffs.cpu().numpy()
    for b, x in enumerate(props):
        r = sf_oracle.solve(op, x, max_iters=8, early_stop=False)
        assert np.abs(coeffs[b] - r.coeffs).max() <= 1e-5 * np.abs(r.coeffs).max(), b
    assert out.eq_err.max().item() <= 1e-8


def test_solve_with_svars_on_the_tensor_core_path():
    """SafetyFilter.solve (svars on: the kernel also keeps the previous iterate, so the tensor-core
    variant runs two slots per CTA) equals solve_batched on the config-2 problem, and its svars are the
    spherical variables of the previous iterate."""
    from dataclasses import replace

    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, sample_proposals
    from paper_2501_19042_b200.scenarios import config_problem
    prob = config_problem(2)
    cfg = SolverConfig(max_iters=40, early_stop=False)
    sf = SafetyFilter(prob, config=cfg)
    props = sample_proposals(prob, sf.basis, 3, seed=5).proposals
    bat = sf.solve_batched(torch.from_numpy(props).cuda(), config=replace(cfg, svars=False), want_prev=True)
    for b in range(3):
        r = sf.solve(props[b])
        assert np.array_equal(r.coeffs, bat.coeffs[b].cpu().numpy())
        assert r.iterations == int(bat.iterations[b])
        sv = sf.svars_of(bat.coeffs_prev[b:b + 1])[0]
        np.testing.assert_array_equal(r.svars.pair_radial, sv.pair_radial)
