"""GPU parity: the sm_100a solve vs the real reference's golden outputs (and the oracle).

Tolerances (written here):
* strict (FP64 terms): coefficients within 1e-9 relative, iteration counts identical;
* lean (FP32 terms, FP64 state; the bench precision): coefficients within 1e-5
  relative of the reference, multipliers within 1e-4 relative, iteration counts
  identical except "borderline" flips where the reference's own residual at the
  stopping iteration lies within 1e-3 relative of tol (F6) -- those are counted;
* hybrid (FP32 screening with guard bands, FP64 targets / residuals / state, FP64 re-evaluation of
  the stop decision near tol): coefficients within 1e-6 relative, iteration counts identical except
  flips where the reference's residual lies within 1e-5 relative of tol;
* feasible verdicts identical.
The antipodal swap is ulp-chaotic (the reference itself warns, test_kernels.py:185-186): its
frozen count (101) depends on glibc's last-ulp trig values, so both precisions are held to the
reference test's behavioural bar instead (converges within 200 iterations, constraints within
1e-2, test_solver.py:218-232).
"""
import numpy as np
import pytest
import torch

from .conftest import SOLVE_CASES, load_golden

pytestmark = pytest.mark.gpu


def _filter_for(case, precision):
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, load_problem
    meta = case["meta"]
    cfg = SolverConfig(precision=precision, svars=False, **meta["config"])
    prob = load_problem(meta["problem"])
    return SafetyFilter(prob, degree=meta["degree"], config=cfg), cfg


def _run(case, precision):
    sf, cfg = _filter_for(case, precision)
    xb = torch.from_numpy(case["proposals"]).cuda()
    kw = {}
    if "xi0" in case:
        kw = dict(xi0=torch.from_numpy(case["xi0"]).cuda(), lam0=torch.from_numpy(case["lam0"]).cuda())
    out = sf.solve_batched(xb, config=cfg, **kw)
    torch.cuda.synchronize()
    return {k: (v.cpu().numpy() if isinstance(v, torch.Tensor) else v) for k, v in vars(out).items()}


def _borderline(ref_hist, its_ref, its_got, tol, band=1e-3):
    k = min(its_ref, its_got) - 1
    return abs(its_ref - its_got) == 1 and abs(ref_hist[k] - tol) <= band * tol


@pytest.mark.parametrize("precision", ["strict", "hybrid", "lean"])
@pytest.mark.parametrize("name", SOLVE_CASES)
def test_solve_matches_reference(name, precision):
    case = load_golden(name)
    out = _run(case, precision)
    tol_res = case["meta"]["config"]["tol_residual"]
    chaotic = name == "antipodal2"
    # head-on swap truncated at k iterations: the robots meet at exactly x = 0, so the sign of the
    # last-ulp round-off there picks one of two mirror-image detours; FP32 positions need not pick the
    # reference's.  Lean is held to the reference test's invariant instead (test_solver.py:241-248).
    mirror = name.startswith("antipodal2_it") and precision != "strict"
    borderline = 0
    for s in range(case["proposals"].shape[0]):
        its_ref, its = int(case["iterations"][s]), int(out["iterations"][s])
        assert out["status"][s] == 0
        if chaotic:
            from paper_2501_19042_b200 import check_coefficients, load_problem
            prob = load_problem(case["meta"]["problem"])
            assert its <= 200 and out["converged"][s]
            assert check_coefficients(out["coeffs"][s], prob, degree=10, tol=1e-2).ok
            continue
        if mirror:
            assert its == its_ref and out["eq_err"][s] <= 1e-8
            np.testing.assert_allclose(out["residual_inf"][s, :its], case["res_inf"][s, :its], rtol=1e-3)
            continue
        if its != its_ref:
            band = 1e-3 if precision == "lean" else 1e-5
            assert precision != "strict" and _borderline(case["res_inf"][s], its_ref, its, tol_res, band), (s, its, its_ref)
            borderline += 1
            continue
        ref_c = case["coeffs"][s]
        scale = max(1.0, np.abs(ref_c).max())
        ctol = {"strict": 1e-9, "hybrid": 1e-6, "lean": 1e-5}[precision]
        err = np.abs(out["coeffs"][s] - ref_c).max() / scale
        assert err <= ctol, (s, err)
        mscale = max(1.0, np.abs(case["multipliers"][s]).max())
        merr = np.abs(out["multipliers"][s] - case["multipliers"][s]).max() / mscale
        assert merr <= ctol * 10, (s, merr)
        hr = case["res_inf"][s, :its]
        hrtol = 1e-6 if precision == "strict" else 5e-2   # hybrid/lean histories: FP32-measured
        np.testing.assert_allclose(out["residual_inf"][s, :its], hr, rtol=hrtol, atol=1e-7)
        np.testing.assert_allclose(out["residual_l2"][s, :its], case["res_l2"][s, :its], rtol=hrtol, atol=1e-7)
        assert bool(out["converged"][s]) == bool(case["converged"][s])
        assert bool(out["feasible"][s]) == bool(case["feasible"][s])
        assert out["eq_err"][s] <= 1e-8
        assert abs(out["displacement"][s] - case["displacement"][s]) <= max(ctol, 1e-9) * max(1.0, case["displacement"][s]) * 10
    assert borderline <= max(1, case["proposals"].shape[0] // 10)


def test_batch_composition_invariance():
    """Results do not depend on batch size, order or launch shape (SPEC determinism)."""
    case = load_golden("crossing4_gen50")
    sf, cfg = _filter_for(case, "lean")
    xb = torch.from_numpy(case["proposals"]).cuda()
    full = sf.solve_batched(xb, config=cfg)
    perm = torch.randperm(xb.shape[0], generator=torch.Generator().manual_seed(0)).cuda()
    shuf = sf.solve_batched(xb[perm], config=cfg, slots_per_block=1, grid=3)
    inv = torch.argsort(perm)
    assert torch.equal(full.coeffs, shuf.coeffs[inv])
    assert torch.equal(full.iterations, shuf.iterations[inv])
    one = sf.solve_batched(xb[7:8], config=cfg)
    assert torch.equal(one.coeffs[0], full.coeffs[7])
