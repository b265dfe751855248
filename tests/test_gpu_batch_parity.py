"""GPU parity on WHOLE batches against the real reference (tests/golden/batch_*.npz).

``batch_cfg3`` / ``batch_cfg4`` are the first 16 / 8 proposals of bench.py's config-3 / config-4 batches
(32 robots H = 100 / 64 robots H = 150), solved by the reference with early stop: converging and
capped samples, pair- and workspace-violating verdicts.

``batch_cfg2`` is the headline workload itself: all 1000 config-2 bench proposals (16 drones,
H = 100, max_iters 500) as the compiled reference solved them -- 998 converged, 765 feasible,
235 converged-but-violating (the pair branch of ``assembly.py:437-487``).  ``batch_ws_tight``
(6 robots squeezed into a tight workspace, tol_residual 0.05) exercises the workspace branch:
26 of its 48 samples end with workspace violations.

Bars (tolerances written here):
* strict (FP64): iteration counts, converged flags and feasible verdicts identical on every
  sample, except flips whose deciding reference quantity lies within 1e-6 (relative residual /
  absolute margin) of its threshold; margins within 1e-9; subset coefficients within 1e-9.
* hybrid (FP32 screening, FP64 values): the strict bar on counts and verdicts; margins within 1e-6,
  subset coefficients within 1e-6 relative.
* lean (FP32 terms): flips are counted and bounded; see DESIGN.md section 5 for the rates.
"""
import pytest

from .batch_parity import compare, run, run_fuzz

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,precision", [
    ("batch_cfg2", "strict"), ("batch_cfg2", "hybrid"), ("batch_ws_tight", "strict"), ("batch_ws_tight", "hybrid"),
    # BASELINE configs 3 / 4 with early stop: 32 robots (K1, two lanes per step; strict does not fit one K1 slot
    # at H = 100 and runs on K1L) and 64 robots, H = 150, max_iters 1000 (K1L)
    ("batch_cfg3", "hybrid"), ("batch_cfg3", "strict"), ("batch_cfg4", "strict"), ("batch_cfg4e", "strict"), ("batch_cfg4", "hybrid"),
    ("batch_cfg4e", "hybrid")])
def test_whole_batch_matches_reference(name, precision):
    g, o = run(name, precision)
    rep = compare(g, o, band=1e-6)
    tol = 1e-9 if precision == "strict" else 1e-6
    assert rep["status_ok"] == rep["batch"]
    assert rep["iter_flip_nonborderline"] == 0, rep["iter_flips"]
    assert rep["verdict_flip_nonborderline"] == 0, rep["verdict_flips"]
    assert rep["iter_flip_count"] + rep["verdict_flip_count"] <= max(1, rep["batch"] // 200)
    assert rep["margin_err_max"] <= tol
    assert rep["viol_count_equal"] == rep["same_iterate"]
    assert rep["coeff_rel_err_max"] is not None and rep["coeff_rel_err_max"] <= tol


@pytest.mark.parametrize("name", ["batch_fuzz", "batch_fuzz_large"])
@pytest.mark.parametrize("precision", ["strict", "hybrid"])
def test_fuzz_scenarios_match_reference(name, precision):
    """``batch_fuzz``: 64 random scenarios x 8 proposals solved by the real reference with early stop -- 2 to 40
    robots (every K1 template incl. the tensor-core n = 16 slot, the two-lane slot and K1L), horizons 20 to 127,
    degrees 7 to 15, rho 0.5 / 1 / 2, tol_residual 1e-3 to 1e-2; 443 converged, 329 feasible, 130 with pair and 12
    with workspace violations, 70 stop at the 300-iteration cap.  ``batch_fuzz_large``: 24 scenarios x 4
    proposals of 17 to 64 robots (two-lane K1, K1L in every precision), horizons 20 to 100.  The strict bar on
    every sample."""
    g, o = run_fuzz(precision, name)
    rep = compare(g, o, band=1e-6)
    tol = 1e-9 if precision == "strict" else 1e-6
    assert rep["status_ok"] == rep["batch"]
    assert rep["iter_flip_nonborderline"] == 0, rep["iter_flips"]
    assert rep["verdict_flip_nonborderline"] == 0, rep["verdict_flips"]
    assert rep["iter_flip_count"] + rep["verdict_flip_count"] <= max(1, rep["batch"] // 200)
    assert rep["margin_err_max"] <= tol
    assert rep["viol_count_equal"] == rep["same_iterate"]
    assert rep["coeff_rel_err_max"] is not None and rep["coeff_rel_err_max"] <= tol


def test_fuzz_scenarios_lean_flip_rate():
    g, o = run_fuzz("lean")
    rep = compare(g, o, band=1e-6)
    assert rep["status_ok"] == rep["batch"]
    assert rep["iter_flip_count"] <= 0.10 * rep["batch"]
    assert abs(rep["feasible_gpu"] - rep["feasible_ref"]) <= 0.05 * rep["batch"]


@pytest.mark.parametrize("name", ["batch_cfg2", "batch_ws_tight"])
def test_lean_whole_batch_flip_rate(name):
    g, o = run(name, "lean")
    rep = compare(g, o, band=1e-6)
    assert rep["status_ok"] == rep["batch"]
    # lean is chaos-sensitive at the 1e-5 level: bound the flip rates
    assert rep["iter_flip_count"] <= 0.10 * rep["batch"]
    assert abs(rep["feasible_gpu"] - rep["feasible_ref"]) <= 0.05 * rep["batch"]
    assert rep["coeff_rel_err_max"] is None or rep["coeff_rel_err_max"] <= 1e-3


def test_worst_first_violation_lists_match_reference():
    """check_coefficients / check_original_constraints list the violations worst first like the reference
    (assembly.py:437-487): the frozen first 8 entries of every violating headline sample, and both branches
    (pairs: batch_cfg2; workspace: batch_ws_tight)."""
    import numpy as np

    from paper_2501_19042_b200 import check_coefficients, coeffs_to_trajectory, check_original_constraints, load_problem
    from paper_2501_19042_b200.basis import build_basis
    for name in ("batch_cfg2", "batch_ws_tight"):
        g, o = run(name, "strict")
        prob = load_problem(g["meta"]["problem"])
        bad = np.nonzero((g["pair_viol"] > 0) | (g["ws_viol"] > 0))[0]
        assert bad.size > 0
        for s in bad[:60]:
            rep = check_coefficients(o["coeffs"][s], prob, degree=g["meta"]["degree"])
            assert rep.pair_violation_count == g["pair_viol"][s] and rep.workspace_violation_count == g["ws_viol"][s]
            for got, ref, width in ((rep.pair_violations, g["pair_list"][s], 3), (rep.workspace_violations, g["ws_list"][s], 2)):
                ref = [r for r in ref if np.isfinite(r).all()]
                assert len(got) >= len(ref)
                for k, r in enumerate(ref):
                    gk = got[k]
                    assert abs(gk[width] - r[width]) <= 1e-9, (name, s, k, gk, r)
                    # identical entry, or a swap of two margins equal to within 1e-9
                    assert tuple(gk[:width]) == tuple(int(v) for v in r[:width]) or \
                        any(abs(gk[width] - rr[width]) <= 1e-9 and tuple(gk[:width]) == tuple(int(v) for v in rr[:width])
                            for rr in ref), (name, s, k, gk, r)
        # the trajectory-level entry point gives the same report
        s = bad[0]
        basis = build_basis(prob.duration, degree=g["meta"]["degree"], samples=prob.horizon_samples)
        rep2 = check_original_constraints(coeffs_to_trajectory(o["coeffs"][s], basis, prob.n), prob)
        rep1 = check_coefficients(o["coeffs"][s], prob, degree=g["meta"]["degree"])
        assert rep2.pair_violation_count == rep1.pair_violation_count
        assert rep2.workspace_violation_count == rep1.workspace_violation_count
        assert [v[:-1] for v in rep2.pair_violations] == [v[:-1] for v in rep1.pair_violations]
