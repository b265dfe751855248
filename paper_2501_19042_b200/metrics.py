"""Evaluation metrics of the reference's `metrics.py`: primal residual, pairwise cosine / diversity,
batch report and its writers.  (`feasible_results` / `feasible_fraction` are in `verdict.py`.)

Diversity definition (as the reference, recorded in every report): flatten each trajectory's sampled
positions (all robots, all axes) into one vector, subtract the batch mean vector, then average the cosine
similarity over all unordered pairs.  Lower means more diverse; identical trajectories are degenerate
after centering and reported as NaN.

The cosine mean runs on the device as an O(count * dim) reduction (`sgsf_pairwise_cosine`): with unit
vectors u_i, sum_{i<j} u_i . u_j = (|sum_i u_i|^2 - sum_i |u_i|^2) / 2, so no Gram matrix is formed.
"""
from __future__ import annotations

import csv
import json
from dataclasses import dataclass, field

import numpy as np
import torch

from . import native
from .errors import TooFewSamples
from .solver import _stream, _to_dev
from .verdict import feasible_results

DIVERSITY_DEFINITION = "centered-position-cosine-mean-over-pairs"


# ------------------------------------------------------------------ reformulated-constraint residual
def spherical_targets(svars, problem):
    """Per-axis targets implied by spherical variables (assembly.py:368-393): pair (3, P, S) and workspace
    (3, n, S), the latter with the centre offset; multiplication order as the reference."""
    lat_r = problem.shape.lateral * svars.pair_radial * np.sin(svars.pair_polar)
    pair = np.stack([lat_r * np.cos(svars.pair_azimuth), lat_r * np.sin(svars.pair_azimuth),
                     problem.shape.vertical * svars.pair_radial * np.cos(svars.pair_polar)])
    lat_rw = problem.workspace.lateral * svars.ws_radial * np.sin(svars.ws_polar)
    ws = np.stack([lat_rw * np.cos(svars.ws_azimuth), lat_rw * np.sin(svars.ws_azimuth),
                   problem.workspace.vertical * svars.ws_radial * np.cos(svars.ws_polar)])
    ws = ws + np.asarray(problem.workspace.center, dtype=float)[:, None, None]
    return pair, ws


def build_spherical_rhs(svars, problem) -> np.ndarray:
    """Flat target vector e in the F layout [pairs (P*S); workspace (n*S)] per axis (assembly.py:396-408)."""
    pair, ws = spherical_targets(svars, problem)
    return np.concatenate([np.concatenate([pair[ax].ravel(), ws[ax].ravel()]) for ax in range(3)])


def primal_residual(coeffs, svars, operator, problem):
    """F xi - e(svars) with its inf and l2 norms (metrics.py:34-41); F xi is evaluated on the device."""
    r = operator.apply(coeffs) - build_spherical_rhs(svars, problem)
    inf = float(np.abs(r).max()) if r.size else 0.0
    return r, inf, float(np.linalg.norm(r))


# ------------------------------------------------------------------ pairwise cosine / diversity
def pairwise_cosine_device(vectors: torch.Tensor, center: bool) -> float:
    """Mean pairwise cosine of the rows of a (count, dim) float64 CUDA tensor (NaN if a row is zero)."""
    V = vectors.to(dtype=torch.float64).contiguous()
    count, dim = int(V.shape[0]), int(V.shape[1])
    if count < 2:
        raise TooFewSamples(f"need at least two vectors for pairwise cosine, got {count}")
    lib = native.load()
    work = torch.empty(int(lib.sgsf_cosine_work_doubles(count, dim)), dtype=torch.float64, device=V.device)
    out = torch.empty(1, dtype=torch.float64, device=V.device)
    native.check(lib.sgsf_pairwise_cosine(count, dim, V.data_ptr(), int(bool(center)), work.data_ptr(),
                                          out.data_ptr(), _stream()), "sgsf_pairwise_cosine")
    return float(out.item())


def mean_pairwise_cosine(vectors) -> float:
    """Mean cosine similarity over all unordered pairs of flat vectors (metrics.py:83-99); NaN when a
    vector is zero."""
    V = np.asarray(vectors, dtype=float)
    if V.ndim != 2:
        V = V.reshape(len(V), -1)
    if V.shape[0] < 2:
        raise TooFewSamples("need at least two vectors for pairwise cosine")
    return pairwise_cosine_device(_to_dev(V), center=False)


def diversity_cosine(trajectories, center: bool = True) -> float:
    """Diversity of a set of trajectories (metrics.py:102-115); `center=False` skips the mean subtraction."""
    trajectories = list(trajectories)
    if len(trajectories) < 2:
        raise TooFewSamples(f"need at least two trajectories, got {len(trajectories)}")
    V = np.stack([np.asarray(t.positions, dtype=float).ravel() for t in trajectories])
    return pairwise_cosine_device(_to_dev(V), center=center)


# ------------------------------------------------------------------ batch report (metrics.py:126-185)
def _nan_to_none(x):
    if x is None:
        return None
    x = float(x)
    return None if np.isnan(x) else x


@dataclass
class BatchReport:
    """Aggregated view of one filtered batch."""

    batch_size: int
    feasible_fraction: float | None
    mean_pairwise_cosine: float | None   # NaN when degenerate, None when < 2 feasible
    feasible_count: int
    converged_count: int
    failed_count: int
    residual_final: list
    displacement: list
    total_time: float
    per_proposal_time: list
    tol: float
    feasible_indices: list = field(default_factory=list)

    def to_jsonable(self) -> dict:
        return {
            "batch_size": self.batch_size,
            "feasible_fraction": _nan_to_none(self.feasible_fraction),
            "mean_pairwise_cosine": _nan_to_none(self.mean_pairwise_cosine),
            "diversity_definition": DIVERSITY_DEFINITION,
            "feasible_count": self.feasible_count,
            "converged_count": self.converged_count,
            "failed_count": self.failed_count,
            "residual_final": [_nan_to_none(r) for r in self.residual_final],
            "displacement": [_nan_to_none(d) for d in self.displacement],
            "total_time": self.total_time,
            "per_proposal_time": self.per_proposal_time,
            "tol": self.tol,
            "feasible_indices": self.feasible_indices,
        }


def build_batch_report(batch, problem, tol: float = 1e-3) -> BatchReport:
    results = batch.results
    feasible = feasible_results(results, problem, tol=tol)
    diversity = diversity_cosine([traj for _, traj in feasible]) if len(feasible) >= 2 else None
    return BatchReport(
        batch_size=len(results),
        feasible_fraction=(len(feasible) / len(results)) if results else None,
        mean_pairwise_cosine=diversity,
        feasible_count=len(feasible),
        converged_count=batch.n_converged,
        failed_count=batch.n_failed,
        residual_final=[r.final_residual_inf for r in results],
        displacement=[r.displacement for r in results],
        total_time=batch.wall_time,
        per_proposal_time=[r.solve_time for r in results],
        tol=tol,
        feasible_indices=[idx for idx, _ in feasible],
    )


def write_csv(path, metadata, header, rows) -> None:
    """CSV with '# key=value' metadata comment lines above the header (metrics.py:212-219)."""
    with open(path, "w", newline="") as fh:
        for key, value in (metadata or {}).items():
            fh.write(f"# {key}={value}\n")
        writer = csv.writer(fh)
        writer.writerow(header)
        writer.writerows(rows)


def save_report_json(report: BatchReport, path, metadata: dict | None = None) -> None:
    """The report as JSON with its metadata (metrics.py:397-401)."""
    doc = {"metadata": dict(metadata or {}), "report": report.to_jsonable()}
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=2)
        fh.write("\n")
