"""Bernstein basis on a uniform time grid (host FP64 constants).

The coefficient vector of a swarm is axis-major, ``(3, n, degree + 1)``
flattened (``basis.py:1-8`` of the reference).  The sampling matrices are
computed once per (degree, samples, duration) in FP64 and uploaded to the
device by the solver; nothing here runs per iteration.
"""
from __future__ import annotations

from dataclasses import dataclass
from math import comb

import numpy as np

from .errors import DegreeTooLow, DimensionMismatch, TooFewSamples

MIN_DEGREE = 5   # six endpoint conditions per axis


def _bernstein_rows(s: np.ndarray, degree: int) -> np.ndarray:
    k = np.arange(degree + 1)
    binom = np.array([float(comb(degree, int(j))) for j in k])
    return binom * s[:, None] ** k * (1.0 - s[:, None]) ** (degree - k)


def bernstein_matrices(degree, samples, duration):
    """(W, Wd, Wdd, time_grid); W is (samples, degree+1), derivatives are d/dt (basis.py:35-69)."""
    if degree < 1:
        raise DegreeTooLow(f"degree must be >= 1, got {degree}")
    if samples < 2:
        raise TooFewSamples(f"need at least 2 samples, got {samples}")
    if not duration > 0:
        raise ValueError(f"duration must be positive, got {duration}")
    grid = np.linspace(0.0, duration, samples)
    s = grid / duration
    W = _bernstein_rows(s, degree)
    low = _bernstein_rows(s, degree - 1)
    Wd = np.zeros_like(W)
    Wd[:, :-1] -= low
    Wd[:, 1:] += low
    Wd *= degree / duration
    Wdd = np.zeros_like(W)
    if degree >= 2:
        low2 = _bernstein_rows(s, degree - 2)
        Wdd[:, :-2] += low2
        Wdd[:, 1:-1] -= 2.0 * low2
        Wdd[:, 2:] += low2
        Wdd *= degree * (degree - 1) / duration ** 2
    return W, Wd, Wdd, grid


@dataclass(frozen=True)
class BasisMatrices:
    value: np.ndarray
    velocity: np.ndarray
    acceleration: np.ndarray
    time_grid: np.ndarray
    duration: float

    @property
    def degree(self) -> int:
        return self.value.shape[1] - 1

    @property
    def samples(self) -> int:
        return self.value.shape[0]


def build_basis(duration, degree=10, samples=50) -> BasisMatrices:
    """Solver basis; rejects degrees that cannot pin p/v/a at both ends (basis.py:91-109)."""
    if degree < MIN_DEGREE:
        raise DegreeTooLow(f"degree {degree} cannot satisfy six endpoint conditions per axis; "
                           f"need at least {MIN_DEGREE}")
    W, Wd, Wdd, grid = bernstein_matrices(degree, samples, duration)
    return BasisMatrices(W, Wd, Wdd, grid, float(duration))


@dataclass(frozen=True)
class Trajectory:
    """Sampled swarm trajectory; arrays are (n, samples, 3)."""

    positions: np.ndarray
    velocities: np.ndarray
    accelerations: np.ndarray
    time_grid: np.ndarray

    @property
    def n(self) -> int:
        return self.positions.shape[0]

    @property
    def samples(self) -> int:
        return self.positions.shape[1]


def coeffs_to_axis_major(coeffs, n, degree) -> np.ndarray:
    xi = np.asarray(coeffs, dtype=float).ravel()
    want = 3 * n * (degree + 1)
    if xi.size != want:
        raise DimensionMismatch(f"coefficient vector has length {xi.size}, expected {want} "
                                f"(n={n}, degree={degree})")
    return xi.reshape(3, n, degree + 1)
