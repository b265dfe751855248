"""GPU parity on WHOLE batches against the real reference (tests/golden/batch_*.npz).

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

from .batch_parity import compare, run

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("precision", ["strict", "hybrid"])
@pytest.mark.parametrize("name", ["batch_cfg2", "batch_ws_tight"])
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


@pytest.mark.parametrize("name", ["batch_cfg2", "batch_ws_tight"])
def test_lean_whole_batch_flip_rate(name):
    g, o = run(name, "lean")
    rep = compare(g, o, band=1e-6)
    assert rep["status_ok"] == rep["batch"]
    # lean is chaos-sensitive at the 1e-5 level: bound the flip rates
    assert rep["iter_flip_count"] <= 0.10 * rep["batch"]
    assert abs(rep["feasible_gpu"] - rep["feasible_ref"]) <= 0.05 * rep["batch"]
    assert rep["coeff_rel_err_max"] is None or rep["coeff_rel_err_max"] <= 1e-3
