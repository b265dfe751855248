"""The reference-side binding (paper_2501_19042_b200/refbind.py, shown verbatim in INTEGRATION.md).

CPU: the document and the module agree; the binding's FP64 precompute runs on the REAL reference's
objects (``swarmfilter`` from oracle/_ref, built by oracle/build_ref.sh; skipped when absent) and equals the
precompute on this package's objects.  GPU: the binding solves through ``sgsf_solve_host`` from a real
``swarmfilter.SafetyFilter`` and from duck-typed objects without a projector, and matches the golden outputs.
"""
import re
import sys
import types
from pathlib import Path

import numpy as np
import pytest

from .conftest import REPO, load_golden

REF = REPO / "oracle" / "_ref"


def _reference():
    if not (REF / "swarmfilter").is_dir():
        pytest.skip("oracle/_ref not built (oracle/build_ref.sh)")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import swarmfilter
    return swarmfilter


def test_integration_doc_shows_the_module_verbatim():
    doc = (REPO / "INTEGRATION.md").read_text()
    blocks = re.findall(r"```python\n(.*?)```", doc, flags=re.S)
    src = (REPO / "paper_2501_19042_b200" / "refbind.py").read_text()
    assert any(b.strip() == src.strip() for b in blocks), "INTEGRATION.md must show refbind.py verbatim"


def test_binding_structs_match_the_header():
    from paper_2501_19042_b200 import native, refbind
    assert [f for f, _ in refbind.Problem._fields_] == [f for f, _ in native.Problem._fields_]
    assert [f for f, _ in refbind.Config._fields_] == [f for f, _ in native.Config._fields_]
    hdr = (REPO / "include" / "sgsf.h").read_text()
    cfg = hdr[hdr.index("typedef struct {\n    int max_iters;"):]
    cfg = cfg[:cfg.index("} sgsf_config_t;")]
    fields = re.findall(r"^\s+(?:int|double)\s+(\w+);", cfg, flags=re.M)
    assert fields == [f for f, _ in refbind.Config._fields_]


def test_precompute_accepts_the_real_reference_objects():
    sfm = _reference()
    from paper_2501_19042_b200 import SafetyFilter, load_problem
    from paper_2501_19042_b200.precompute import device_constants
    from paper_2501_19042_b200.scenarios import config_doc
    doc = config_doc(2)
    ref = sfm.SafetyFilter(sfm.load_problem(doc), degree=10)
    assert not hasattr(ref.equality, "projector")
    k_ref = device_constants(ref.problem, ref.basis, ref.equality, 1.0)
    ours = SafetyFilter(load_problem(doc), degree=10)
    k_own = device_constants(ours.problem, ours.basis, ours.equality, 1.0)
    for f in ("W", "Wd", "Wdd", "B", "rhs", "PBt", "Km11", "Kd11", "Mm", "Md", "cconst", "center"):
        a, b = getattr(k_ref, f), getattr(k_own, f)
        assert a.shape == b.shape, f
        np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-14, err_msg=f)


@pytest.mark.gpu
def test_binding_solves_from_the_real_reference_filter():
    sfm = _reference()
    from paper_2501_19042_b200.refbind import batch_solve_b200
    case = load_golden("swarm16_cfg2")
    meta = case["meta"]
    ref = sfm.SafetyFilter(sfm.load_problem(meta["problem"]), degree=meta["degree"],
                           config=sfm.SolverConfig(**meta["config"]))
    out = batch_solve_b200(ref, case["proposals"], ref.config)
    assert (out["status"] == 0).all()
    np.testing.assert_array_equal(out["iterations"], case["iterations"])
    np.testing.assert_array_equal(out["converged"].astype(bool), case["converged"])
    np.testing.assert_array_equal(out["feasible"].astype(bool), case["feasible"])
    scale = np.abs(case["coeffs"]).max()
    assert np.abs(out["coeffs"] - case["coeffs"]).max() <= 1e-6 * scale


@pytest.mark.gpu
def test_binding_on_duck_typed_objects_without_projector():
    """The binding needs only the reference's attribute names: an equality object with `block` and
    `rhs_axes` alone (no projector) works."""
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, load_problem
    from paper_2501_19042_b200.refbind import batch_solve_b200
    case = load_golden("crossing4_cfg1")
    meta = case["meta"]
    own = SafetyFilter(load_problem(meta["problem"]), degree=meta["degree"])
    eq = types.SimpleNamespace(block=own.equality.block, rhs_axes=own.equality.rhs_axes)
    duck = types.SimpleNamespace(problem=own.problem, basis=own.basis, equality=eq)
    cfg = SolverConfig(**meta["config"])
    out = batch_solve_b200(duck, case["proposals"], cfg, precision="strict")
    np.testing.assert_array_equal(out["iterations"], case["iterations"])
    scale = np.abs(case["coeffs"]).max()
    assert np.abs(out["coeffs"] - case["coeffs"]).max() <= 1e-9 * scale
