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
from pathlib import Path

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


# ------------------------------------------------------------------ benchmark sweeps (metrics.py:188-395)
@dataclass(frozen=True)
class BenchmarkGrid:
    """Axes of the benchmark sweeps (fig5a/5b: batch sizes; fig6: batch sizes and iteration counts;
    fig7: init strategies)."""

    batch_sizes: tuple = (1, 10, 50)
    iteration_counts: tuple = (50, 100, 200, 400)
    strategies: tuple = ("zero", "projected", "warmstart")
    timing_batch: int = 10
    trace_iters: int = 200
    seed: int = 0
    spread: float = 0.25

    def __post_init__(self):
        unknown = sorted(set(self.strategies) - {"zero", "projected", "warmstart"})
        if unknown:
            raise ValueError(f"unknown init strategies {unknown}; choose from ['projected', 'warmstart', 'zero']")
        if not self.batch_sizes or min(self.batch_sizes) < 1:
            raise ValueError(f"batch sizes must be >= 1, got {self.batch_sizes}")
        if not self.iteration_counts or min(self.iteration_counts) < 1:
            raise ValueError(f"iteration counts must be >= 1, got {self.iteration_counts}")


_PLOTS = {
    "fig5a": ("feasible fraction vs batch size",
              "set xlabel 'batch size'\nset ylabel 'feasible fraction'\nset yrange [0:1.05]\n"
              "plot 'fig5a.csv' using 2:3 with linespoints title 'feasible fraction'\n"),
    "fig5b": ("mean pairwise cosine of feasible solutions",
              "set xlabel 'row'\nset ylabel 'mean pairwise cosine'\n"
              "plot 'fig5b.csv' using 0:2 with linespoints title 'cosine'\n"),
    "fig6": ("wall-clock time scaling",
             "set xlabel 'iterations'\nset ylabel 'seconds'\n"
             "plot 'fig6.csv' using 2:3 with linespoints title 'batch time'\n"),
    "fig7": ("residual vs iteration per init strategy",
             "set xlabel 'iteration'\nset ylabel 'inf-norm residual'\nset logscale y\n"
             "plot for [s in strategies] 'fig7.csv' using (strcol(1) eq s ? $2 : 1/0):3 with lines title s\n"),
}


def _fmt(x) -> str:
    return "nan" if x is None else repr(float(x))


def _gnuplot(out_dir: Path, name: str, strategies=None) -> Path:
    title, body = _PLOTS[name]
    head = ["#!/usr/bin/env gnuplot", "set datafile separator ','", "set datafile commentschars '#'",
            "set key autotitle columnhead", f"set title '{title}'", "set terminal pngcairo size 800,600",
            f"set output '{name}.png'"]
    if name == "fig7" and strategies is not None:
        head.append(f"strategies = '{' '.join(strategies)}'")
    path = out_dir / f"{name}.gp"
    path.write_text("\n".join(head + [body]))
    return path


def benchmark(problem, grid: BenchmarkGrid, out_dir, config=None, degree: int = 10, threads: int = 1,
              metadata: dict | None = None, tol_check: float = 1e-3) -> dict:
    """The reference's three sweeps (metrics.py:266-389), on the device solver: feasibility and diversity
    vs batch size (fig5a, fig5b), wall clock vs batch size and iteration count with early stop off (fig6),
    and the residual trace of one proposal per init strategy (fig7).  Returns the output paths."""
    import time
    from dataclasses import replace

    from .proposals import WarmStart, sample_proposals
    from .solver import SafetyFilter, SolverConfig

    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    cfg = config if config is not None else SolverConfig()
    sf = SafetyFilter(problem, degree=degree, config=cfg)
    meta = dict(metadata or {})
    meta.setdefault("seed", grid.seed)
    meta.setdefault("diversity_definition", DIVERSITY_DEFINITION)
    props_of = lambda count: sample_proposals(problem, sf.basis, count, seed=grid.seed, spread=grid.spread).proposals
    paths = {}

    rows_a, rows_b = [], []
    for batch_size in grid.batch_sizes:
        report = build_batch_report(sf.batch_solve(props_of(batch_size), threads=threads), problem, tol=tol_check)
        rows_a.append([problem.n, batch_size, _fmt(report.feasible_fraction)])
        rows_b.append([problem.n, _fmt(report.mean_pairwise_cosine)])
    paths["fig5a"], paths["fig5b"] = out_dir / "fig5a.csv", out_dir / "fig5b.csv"
    write_csv(paths["fig5a"], meta, ["n", "batch", "feasible_fraction"], rows_a)
    write_csv(paths["fig5b"], meta, ["n", "mean_pairwise_cosine"], rows_b)

    fixed = replace(cfg, early_stop=False)
    rows_6 = []
    timed = [(b, props_of(b), fixed) for b in grid.batch_sizes]
    timed += [(grid.timing_batch, props_of(grid.timing_batch), replace(fixed, max_iters=it))
              for it in grid.iteration_counts]
    for batch_size, props, c in timed:
        t0 = time.perf_counter()
        sf.batch_solve(props, threads=threads, config=c)
        dt = time.perf_counter() - t0
        rows_6.append([batch_size, c.max_iters, _fmt(dt), _fmt(dt / batch_size)])
    paths["fig6"] = out_dir / "fig6.csv"
    write_csv(paths["fig6"], meta, ["batch", "iters", "seconds", "seconds_per_proposal"], rows_6)

    proposal = props_of(1)[0]
    trace = replace(fixed, max_iters=grid.trace_iters)
    inits = {"zero": (np.zeros(proposal.size), np.zeros(proposal.size)), "projected": None}
    if "warmstart" in grid.strategies:
        prior = sf.solve(proposal, config=trace)
        inits["warmstart"] = WarmStart(xi0=prior.coeffs, lambda0=prior.multipliers)
    rows_7 = []
    for strategy in grid.strategies:
        res = sf.solve(proposal, init=inits[strategy], config=trace)
        rows_7 += [[strategy, k + 1, _fmt(float(res.residual_inf[k]))] for k in range(res.iterations)]
    paths["fig7"] = out_dir / "fig7.csv"
    write_csv(paths["fig7"], meta, ["strategy", "iter", "res_inf"], rows_7)

    for name in ("fig5a", "fig5b", "fig6", "fig7"):
        paths[f"{name}_plot"] = _gnuplot(out_dir, name, grid.strategies if name == "fig7" else None)
    return paths
