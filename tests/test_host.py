"""CPU tests of the host side: problem types, sampler, precompute, the
kernel reformulation (numpy statement of the device algorithm) and the C-ABI
library surface.  No GPU needed."""
import ctypes
import json
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import sf_oracle as so
from paper_2501_19042_b200 import (
    DimensionMismatch,
    ProblemValidationError,
    SchemaMismatch,
    SolverConfig,
    build_basis,
    build_equality,
    device_constants,
    load_problem,
    project_to_boundary,
    sample_proposals,
    straight_line_coeffs,
)
from paper_2501_19042_b200.precompute import decoupled_step_host
from paper_2501_19042_b200.scenarios import CROSSING4, config_problem, random_swarm_doc

from .conftest import REPO, load_golden
from .kernel_spec import spec_solve


def _setup(doc, degree=10, rho=1.0):
    prob = load_problem(doc)
    basis = build_basis(prob.duration, degree=degree, samples=prob.horizon_samples)
    eq = build_equality(prob, basis)
    return prob, basis, eq, device_constants(prob, basis, eq, rho)


# ------------------------------------------------------------------ problem / inputs
def test_load_problem_schema_errors():
    with pytest.raises(SchemaMismatch):
        load_problem({"n": 1})
    bad = json.loads(json.dumps(CROSSING4))
    bad["boundary"][1]["goal"]["p"] = bad["boundary"][0]["goal"]["p"]   # goal collision
    with pytest.raises(ProblemValidationError, match="goal positions violate"):
        load_problem(bad)


def test_solver_config_validation():
    for kw in ({"rho": 0.0}, {"max_iters": 0}, {"tol_residual": 0.0}, {"tol_eq": -1.0}, {"precision": "fp16"}):
        with pytest.raises(ValueError):
            SolverConfig(**kw)


def test_sampler_reproduces_reference_proposals():
    """Same RNG stream and arithmetic as proposals.py:83-129 -> same inputs as the golden run."""
    case = load_golden("crossing4_cfg1")
    prob = load_problem(case["meta"]["problem"])
    basis = build_basis(prob.duration, 10, prob.horizon_samples)
    props = sample_proposals(prob, basis, 8, seed=0).proposals
    np.testing.assert_allclose(props, case["proposals"], atol=1e-12)
    case16 = load_golden("swarm16_cfg2")
    p16 = load_problem(case16["meta"]["problem"])
    b16 = build_basis(p16.duration, 10, p16.horizon_samples)
    np.testing.assert_allclose(sample_proposals(p16, b16, 4, seed=0).proposals, case16["proposals"], atol=1e-12)


def test_config_scenarios_are_valid_and_seeded():
    assert config_problem(1).n == 4
    p2 = config_problem(2)
    assert (p2.n, p2.horizon_samples) == (16, 101)
    assert random_swarm_doc(16, 100, seed=2) == random_swarm_doc(16, 100, seed=2)


def test_boundary_projection_matches_oracle_and_is_idempotent():
    st = load_golden("steps_small")
    prob, basis, eq, _ = _setup(json.loads(str(st["problem"])), degree=5)
    for c in range(st["xi"].shape[0]):
        x = project_to_boundary(st["xi"][c], eq)
        np.testing.assert_allclose(x, st["projected"][c], atol=1e-12)
        np.testing.assert_allclose(project_to_boundary(x, eq), x, atol=1e-12)
        assert np.abs(eq.residual(x)).max() <= 1e-12


# ------------------------------------------------------------------ decoupled KKT (precompute)
@pytest.mark.parametrize("n,degree,rho", [(1, 10, 1.0), (3, 5, 1.7), (4, 10, 0.3), (16, 10, 1.0)])
def test_decoupled_kkt_equals_dense_lu(n, degree, rho):
    """The per-axis 17n saddle system splits exactly into a mean and a deviation KKT
    (precompute.py); the device xi-step in residual-identity form must equal the
    reference's dense LU coefficient step (assembly.py:186-219)."""
    doc = CROSSING4 if n == 4 else random_swarm_doc(n, 20, seed=n)
    prob, basis, eq, k = _setup(doc, degree=degree, rho=rho)
    oprob = so.make_problem(doc, degree=degree)
    rng = np.random.default_rng(7)
    dim = k.cconst.size
    C = rng.standard_normal(dim)
    lam = rng.standard_normal(dim)
    lam_new = rng.standard_normal(dim)
    xbar = rng.standard_normal(dim)
    # eta of the reference for targets e with F^T e = F^T F C - (lam - lam_new)/rho
    FtF_C = so.transpose_flat(oprob, so.apply_F(oprob, C))
    eta = rho * FtF_C - (lam - lam_new) + lam_new + xbar
    ref = so.kkt_solve(oprob, rho, eta.reshape(3, -1), tol_eq=1e-8).ravel()
    got = decoupled_step_host(k, C, lam_new, lam, xbar)
    np.testing.assert_allclose(got, ref, atol=1e-9 * max(1.0, np.abs(ref).max()))
    assert np.abs(eq.residual(got)).max() <= 1e-10


# ------------------------------------------------------------------ the kernel's algorithm on CPU
@pytest.mark.parametrize("name", ["asym2", "crossing4_cfg1", "tri_deg7", "single1", "parallel2"])
@pytest.mark.parametrize("term", [np.float64, np.float32])
def test_kernel_algorithm_statement_matches_reference(name, term):
    """tests/kernel_spec.py (trig-free projection + FP64 fallback on zero components,
    residual identity, decoupled xi-step, exit residual against recomputed old
    targets) reproduces the reference: FP64 to 1e-12, FP32 terms to 1e-6."""
    case = load_golden(name)
    meta = case["meta"]
    prob, basis, eq, k = _setup(meta["problem"], degree=meta["degree"], rho=meta["config"]["rho"])
    cfg = meta["config"]
    for s, xb in enumerate(case["proposals"]):
        r = spec_solve(k, xb, max_iters=cfg["max_iters"], tol_residual=cfg["tol_residual"],
                       early_stop=cfg["early_stop"], term=term)
        assert r["iterations"] == int(case["iterations"][s])
        scale = max(1.0, np.abs(case["coeffs"][s]).max())
        tol = 1e-12 if term is np.float64 else 1e-6
        assert np.abs(r["coeffs"] - case["coeffs"][s]).max() / scale <= tol


def test_quiet_identities():
    """Closed forms the kernel uses for time steps with every term interior:
    max_{i<j} |a_i - a_j| = max a - min a and sum_{i<j} (a_i - a_j)^2 = (n+1) S2 - S1^2 - S2."""
    rng = np.random.default_rng(3)
    for n in (1, 2, 7, 16):
        a = rng.standard_normal(n)
        pi, pj = np.triu_indices(n, 1)
        pair_max = np.abs(a[pi] - a[pj]).max() if n > 1 else 0.0
        assert np.isclose(pair_max, a.max() - a.min())
        total = np.sum((a[pi] - a[pj]) ** 2) + np.sum(a ** 2)
        assert np.isclose(total, (n + 1) * np.sum(a ** 2) - np.sum(a) ** 2)


# ------------------------------------------------------------------ C ABI surface
def test_library_exports_every_declared_symbol():
    from paper_2501_19042_b200 import native
    header = (REPO / "include" / "sgsf.h").read_text()
    declared = set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(sgsf_\w+)\s*\(", header, flags=re.M))
    assert declared, "no declarations parsed"
    lib = ctypes.CDLL(str(native.LIB_PATH))
    for name in declared:
        assert hasattr(lib, name), name
    assert set(native.EXPORTS) == declared
    assert native.load().sgsf_max_robots() >= 16


def test_product_path_has_no_cpu_fallback():
    """The package never imports the oracle, and refuses to solve without CUDA."""
    pkg = REPO / "paper_2501_19042_b200"
    for f in pkg.rglob("*.py"):
        assert "oracle" not in f.read_text().replace("oracle/", ""), f
    import torch
    if not torch.cuda.is_available():
        from paper_2501_19042_b200 import SafetyFilter
        sf = SafetyFilter(load_problem(CROSSING4))
        with pytest.raises(Exception, match="CUDA"):
            sf.solve(straight_line_coeffs(sf.problem, sf.basis))


def test_bench_flop_formula():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", REPO / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    # config 2 (n=16, S=101, m1=11) -> 692,376 FLOP per sample-iteration
    assert bench.flop_per_si(16, 101, 11) == 692376
    assert bench.flop_per_si(4, 51, 11) == 50802
