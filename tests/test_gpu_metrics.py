"""Metrics on the GPU (metrics.py of the reference): the reference's own metric tests restated, and the
device cosine reduction against the reference's Gram-matrix formula (oracle)."""
import math

import numpy as np
import pytest
import torch

from oracle import sf_oracle

pytestmark = pytest.mark.gpu


def traj_from_positions(pos):
    from paper_2501_19042_b200.basis import Trajectory
    pos = np.asarray(pos, dtype=float)
    zeros = np.zeros_like(pos)
    return Trajectory(positions=pos, velocities=zeros, accelerations=zeros,
                      time_grid=np.arange(pos.shape[1], dtype=float))


class TestCosine:   # test_metrics.py:140-185
    def test_duplicates_uncentered_is_one(self):
        from paper_2501_19042_b200 import mean_pairwise_cosine
        assert mean_pairwise_cosine([[1.0, 2.0, 3.0]] * 3) == pytest.approx(1.0, abs=1e-15)

    def test_duplicates_centered_is_nan(self):
        from paper_2501_19042_b200 import diversity_cosine
        assert math.isnan(diversity_cosine([traj_from_positions([[(1.0, 2.0, 3.0)]])] * 3))

    def test_orthogonal_is_zero(self):
        from paper_2501_19042_b200 import mean_pairwise_cosine
        assert mean_pairwise_cosine([[1.0, 0.0], [0.0, 1.0]]) == 0.0

    def test_analytic_inverse_sqrt2(self):
        from paper_2501_19042_b200 import mean_pairwise_cosine
        assert mean_pairwise_cosine([[1.0, 0.0], [1.0, 1.0]]) == pytest.approx(1.0 / np.sqrt(2.0), abs=1e-12)

    def test_diversity_orthogonal_after_centering(self):
        from paper_2501_19042_b200 import diversity_cosine
        base = np.zeros((3, 1, 2, 3))
        base[0, 0, 0, 0] = base[1, 0, 0, 1] = base[2, 0, 0, 2] = 1.0
        assert diversity_cosine([traj_from_positions(b) for b in base]) == pytest.approx(-0.5, abs=1e-12)

    def test_too_few_vectors(self):
        from paper_2501_19042_b200 import TooFewSamples, diversity_cosine, mean_pairwise_cosine
        with pytest.raises(TooFewSamples):
            mean_pairwise_cosine([[1.0, 0.0]])
        with pytest.raises(TooFewSamples):
            diversity_cosine([traj_from_positions([[(1.0, 0.0, 0.0)]])])

    @pytest.mark.parametrize("count,dim,center", [(2, 3, False), (7, 50, True), (300, 4848, True), (1000, 97, False)])
    def test_matches_gram_formula(self, count, dim, center):
        from paper_2501_19042_b200.metrics import pairwise_cosine_device
        rng = np.random.default_rng(count + dim)
        V = rng.standard_normal((count, dim)) + 0.3
        ref = sf_oracle.mean_pairwise_cosine(V - V.mean(axis=0) if center else V)
        got = pairwise_cosine_device(torch.from_numpy(V).cuda(), center)
        assert got == pytest.approx(ref, abs=1e-13)

    def test_translation_invariance(self):
        from paper_2501_19042_b200 import diversity_cosine
        pos = np.random.default_rng(61).standard_normal((4, 2, 5, 3))
        base = diversity_cosine([traj_from_positions(p) for p in pos])
        moved = diversity_cosine([traj_from_positions(p + np.array([50.0, -3.0, 7.0])) for p in pos])
        assert moved == pytest.approx(base, abs=1e-9)


def test_primal_residual_equals_last_history_entry():
    """test_metrics.py:71-78: the residual of the returned iterate against its spherical variables equals
    the last history entry -- here from the device F and the reference target formula."""
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, primal_residual, straight_line_coeffs
    from paper_2501_19042_b200.problem import load_problem
    doc = {"n": 2, "H": 20, "T": 2.0, "a": 0.6, "b": 0.4,
           "workspace": {"center": [0.0, 0.0, 1.0], "a_w": 5.0, "b_w": 3.0},
           "boundary": [{"start": {"p": [1.5, 0.3, 1.0]}, "goal": {"p": [-1.5, 0.1, 1.1]}},
                        {"start": {"p": [-1.5, -0.2, 0.9]}, "goal": {"p": [1.5, -0.3, 1.0]}}]}
    prob = load_problem(doc)
    sf = SafetyFilter(prob, degree=10, config=SolverConfig(precision="strict"))
    res = sf.solve(straight_line_coeffs(prob, sf.basis))
    r, inf, l2 = primal_residual(res.coeffs, res.svars, sf.operator, prob)
    assert r.shape == (sf.operator.rows,)
    assert abs(inf - res.residual_inf[-1]) <= 1e-9
    assert abs(l2 - res.residual_l2[-1]) <= 1e-9


def test_batch_report_and_writers(tmp_path):
    """test_metrics.py:190-230: report fields on a real batch, JSON and CSV writers; the diversity of the
    feasible set equals the oracle's Gram-matrix formula on the same trajectories."""
    import json
    from paper_2501_19042_b200 import (SafetyFilter, build_batch_report, feasible_results, sample_proposals,
                                       save_report_json, write_csv)
    from paper_2501_19042_b200.scenarios import config_problem
    prob = config_problem(1)
    sf = SafetyFilter(prob, degree=10)
    batch = sf.batch_solve(sample_proposals(prob, sf.basis, 8, seed=2).proposals)
    report = build_batch_report(batch, prob)
    assert report.batch_size == 8 and report.failed_count == 0
    assert report.feasible_count == len(report.feasible_indices)
    feas = feasible_results(batch.results, prob)
    ref = sf_oracle.diversity_cosine([t.positions for _, t in feas])
    assert report.mean_pairwise_cosine == pytest.approx(ref, abs=1e-12)
    save_report_json(report, tmp_path / "r.json", {"seed": 2})
    doc = json.loads((tmp_path / "r.json").read_text())
    assert doc["metadata"] == {"seed": 2} and doc["report"]["diversity_definition"].startswith("centered")
    write_csv(tmp_path / "x.csv", {"k": 1}, ["a", "b"], [[1, 2], [3, 4]])
    assert (tmp_path / "x.csv").read_text().splitlines() == ["# k=1", "a,b", "1,2", "3,4"]


def test_benchmark_sweep_outputs(tmp_path):
    """metrics.benchmark (test_metrics.py:230-): the four CSVs and plot scripts, deterministic fig5 rows,
    one fig7 trace per strategy."""
    import csv as _csv
    from paper_2501_19042_b200 import BenchmarkGrid, SolverConfig, benchmark
    from paper_2501_19042_b200.scenarios import config_problem
    prob = config_problem(1)
    grid = BenchmarkGrid(batch_sizes=(2, 4), iteration_counts=(5, 10), timing_batch=2, trace_iters=20)
    paths = benchmark(prob, grid, tmp_path, config=SolverConfig(max_iters=100))
    for name in ("fig5a", "fig5b", "fig6", "fig7"):
        assert paths[name].exists() and paths[f"{name}_plot"].exists()
    rows = [r for r in _csv.reader(open(paths["fig7"])) if r and not r[0].startswith("#")]
    assert rows[0] == ["strategy", "iter", "res_inf"]
    assert {r[0] for r in rows[1:]} == {"zero", "projected", "warmstart"}
    again = benchmark(prob, grid, tmp_path / "b", config=SolverConfig(max_iters=100))
    assert open(paths["fig5a"]).read() == open(again["fig5a"]).read()
    with pytest.raises(ValueError):
        BenchmarkGrid(strategies=("bogus",))
