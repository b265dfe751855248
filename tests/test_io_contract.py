"""Proposal / warm-start JSON I/O and the report metrics, against the reference's own schema and pins.

CPU (reference from oracle/_ref; skipped when it is absent): files written by this package load in the
reference and the reverse, with identical arrays and documents (proposals.py:136-272).  GPU: the warm start
from saved solutions converges in [1, 1, 1, 1] iterations (test_cli.py:208-233) and the batch report's
diversity reproduces the reference's pinned cosine -0.019914830342448342 +- 1e-9 on `generate crossing4`
(test_cli.py:55-66).
"""
import json
import sys

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


def _crossing4(sfm=None):
    from paper_2501_19042_b200 import SafetyFilter, load_problem
    from paper_2501_19042_b200.scenarios import CROSSING4
    prob = load_problem(CROSSING4)
    return prob, SafetyFilter(prob, degree=10)


def test_proposal_files_round_trip_with_the_reference(tmp_path):
    sfm = _reference()
    from paper_2501_19042_b200 import load_proposals, sample_proposals, save_proposals
    from paper_2501_19042_b200.scenarios import CROSSING4
    prob, sf = _crossing4()
    rprob = sfm.load_problem(CROSSING4)
    ours = sample_proposals(prob, sf.basis, 4, seed=7)
    theirs = sfm.sample_proposals(rprob, sfm.SafetyFilter(rprob, degree=10).basis, 4, seed=7)
    # same sampler draws; the boundary projection's arithmetic differs in the last bits
    np.testing.assert_allclose(ours.proposals, theirs.proposals, rtol=0, atol=1e-13)
    from paper_2501_19042_b200.proposals import ProposalBatch
    ours = ProposalBatch(theirs.proposals.copy(), theirs.provenance, theirs.seed)   # the same batch, both writers
    save_proposals(ours, tmp_path / "ours.json", problem=prob)
    sfm.save_proposals(theirs, tmp_path / "theirs.json", problem=rprob)
    assert json.loads((tmp_path / "ours.json").read_text()) == json.loads((tmp_path / "theirs.json").read_text())
    a = sfm.load_proposals(tmp_path / "ours.json", rprob)      # the reference reads ours
    b = load_proposals(tmp_path / "theirs.json", prob)         # we read the reference's
    np.testing.assert_array_equal(a.proposals, ours.proposals)
    np.testing.assert_array_equal(b.proposals, theirs.proposals)
    assert (a.provenance, a.seed, a.projected_on_load) == (b.provenance, b.seed, b.projected_on_load)


def test_warmstart_files_round_trip_with_the_reference(tmp_path):
    sfm = _reference()
    from paper_2501_19042_b200 import WarmStart, load_warmstart, save_warmstarts
    from paper_2501_19042_b200.scenarios import CROSSING4
    prob, sf = _crossing4()
    rprob = sfm.load_problem(CROSSING4)
    rng = np.random.default_rng(0)
    xi, lam = rng.normal(size=(3, sf.coeff_dim)), rng.normal(size=(3, sf.coeff_dim))
    save_warmstarts([WarmStart(x, l) for x, l in zip(xi, lam)], tmp_path / "ours.json", problem=prob)
    sfm.save_warmstarts([sfm.WarmStart(x, l) for x, l in zip(xi, lam)], tmp_path / "theirs.json", problem=rprob)
    assert json.loads((tmp_path / "ours.json").read_text()) == json.loads((tmp_path / "theirs.json").read_text())
    for starts in (sfm.load_warmstart(tmp_path / "ours.json", rprob), load_warmstart(tmp_path / "theirs.json", prob)):
        np.testing.assert_array_equal(np.stack([w.xi0 for w in starts]), xi)
        np.testing.assert_array_equal(np.stack([w.lambda0 for w in starts]), lam)


def test_warmstart_file_validation_matches_the_reference(tmp_path):
    """A warm-start file for another swarm size is rejected by both with DimensionMismatch."""
    sfm = _reference()
    from paper_2501_19042_b200 import WarmStart, load_warmstart, save_warmstarts
    from paper_2501_19042_b200.errors import DimensionMismatch
    from paper_2501_19042_b200.scenarios import CROSSING4, config_doc
    from paper_2501_19042_b200 import load_problem
    big = load_problem(config_doc(2))
    dim = 3 * big.n * 11
    save_warmstarts([WarmStart(np.zeros(dim), np.zeros(dim))], tmp_path / "w.json", problem=big)
    with pytest.raises(DimensionMismatch):
        load_warmstart(tmp_path / "w.json", load_problem(CROSSING4))
    with pytest.raises(sfm.errors.DimensionMismatch):
        sfm.load_warmstart(tmp_path / "w.json", sfm.load_problem(CROSSING4))


@pytest.mark.gpu
def test_warm_start_from_saved_solutions_converges_immediately(tmp_path):
    """test_cli.py:208-233: filter 4 sampled crossing4 proposals, save the solutions as warm starts, filter
    again from them: [1, 1, 1, 1] iterations, fewer than cold."""
    from paper_2501_19042_b200 import (WarmStart, feasible_results, load_proposals, load_warmstart,
                                       sample_proposals, save_proposals, save_warmstarts)
    prob, sf = _crossing4()
    save_proposals(sample_proposals(prob, sf.basis, 4, seed=7), tmp_path / "c4.json", problem=prob)
    props = load_proposals(tmp_path / "c4.json", prob).proposals
    cold = sf.batch_solve(props)
    feas = feasible_results(cold.results, prob)
    starts = [WarmStart(cold.results[i].coeffs, cold.results[i].multipliers) for i, _ in feas]
    save_warmstarts(starts, tmp_path / "solutions.json", problem=prob)
    warm = sf.batch_solve(props, inits=load_warmstart(tmp_path / "solutions.json", prob))
    its_cold = [r.iterations for r in cold.results]
    its_warm = [r.iterations for r in warm.results]
    assert len(its_warm) == 4 and sum(its_warm) < sum(its_cold)
    assert its_warm == [1, 1, 1, 1]


@pytest.mark.gpu
def test_report_diversity_reproduces_the_reference_pin():
    """`generate crossing4` (50 proposals, seed 0, 200 iterations): feasible fraction 1.0 and mean pairwise
    cosine -0.019914830342448342 +- 1e-9 (test_cli.py:55-66), via the batch report on the device."""
    from paper_2501_19042_b200 import SolverConfig, build_batch_report
    case = load_golden("crossing4_gen50")
    prob, sf = _crossing4()
    batch = sf.batch_solve(list(case["proposals"]), config=SolverConfig(**case["meta"]["config"]))
    np.testing.assert_array_equal([r.iterations for r in batch.results], case["iterations"])
    rep = build_batch_report(batch, prob)
    assert rep.feasible_fraction == 1.0 and rep.failed_count == 0
    assert rep.mean_pairwise_cosine == pytest.approx(-0.019914830342448342, abs=1e-9)
