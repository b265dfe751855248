"""Seeded synthetic scenarios for the benchmark configurations.

The reference ships one scenario (``scenarios/crossing4.json``: n=4, H=50).
BASELINE configs 2-4 (n = 16 / 32 / 64) have none, so this generator makes
them reproducibly: robot spheroid a=0.6, b=0.4; workspace centred
at (0, 0, 1) with a_w = max(5, 1.25 sqrt(n)), b_w = 3; starts and goals drawn
uniformly in the workspace's bounding box, kept when inside the 0.8-scaled
workspace and at normalised clearance > 1.2 from every point already accepted
in the same set; T = 0.1 H seconds; endpoint velocity/acceleration zero.
Exact antipodal rings are avoided on purpose: they are ulp-chaotic.
"""
from __future__ import annotations

import math

import numpy as np

from .problem import load_problem

CROSSING4 = {
    "n": 4, "H": 50, "T": 5.0, "a": 0.6, "b": 0.4,
    "workspace": {"center": [0.0, 0.0, 1.0], "a_w": 5.0, "b_w": 3.0},
    "boundary": [
        {"start": {"p": [2.0, 0.0, 1.0]}, "goal": {"p": [-2.0, 0.0, 1.0]}},
        {"start": {"p": [0.0, 2.0, 1.0]}, "goal": {"p": [0.0, -2.0, 1.0]}},
        {"start": {"p": [-2.0, 0.0, 1.0]}, "goal": {"p": [2.0, 0.0, 1.0]}},
        {"start": {"p": [0.0, -2.0, 1.0]}, "goal": {"p": [0.0, 2.0, 1.0]}},
    ],
}


def _draw_points(rng, n, a, b, a_w, b_w, center, clearance):
    pts = []
    while len(pts) < n:
        p = np.array([rng.uniform(-a_w, a_w), rng.uniform(-a_w, a_w),
                      rng.uniform(center[2] - b_w, center[2] + b_w)])
        d = p - center
        if (d[0] ** 2 + d[1] ** 2) / (0.8 * a_w) ** 2 + d[2] ** 2 / (0.8 * b_w) ** 2 > 1.0:
            continue
        ok = True
        for q in pts:
            e = p - q
            if math.sqrt((e[0] ** 2 + e[1] ** 2) / a ** 2 + e[2] ** 2 / b ** 2) <= clearance:
                ok = False
                break
        if ok:
            pts.append(p)
    return pts


def random_swarm_doc(n: int, horizon: int, seed: int, a: float = 0.6, b: float = 0.4,
                     clearance: float = 1.2) -> dict:
    """Reference-schema problem dict for n robots with random start/goal sets."""
    a_w = max(5.0, 1.25 * math.sqrt(n))
    b_w = 3.0
    center = np.array([0.0, 0.0, 1.0])
    rng = np.random.default_rng(seed)
    starts = _draw_points(rng, n, a, b, a_w, b_w, center, clearance)
    goals = _draw_points(rng, n, a, b, a_w, b_w, center, clearance)
    return {
        "n": n, "H": horizon, "T": 0.1 * horizon, "a": a, "b": b,
        "workspace": {"center": center.tolist(), "a_w": a_w, "b_w": b_w},
        "boundary": [{"start": {"p": [float(x) for x in s]}, "goal": {"p": [float(x) for x in g]}}
                     for s, g in zip(starts, goals)],
    }


def local_swarm_doc(n: int, horizon: int, seed: int, travel: float, a: float = 0.6, b: float = 0.4,
                    clearance: float = 1.2) -> dict:
    """Like random_swarm_doc, but every goal lies `travel` away from its robot's start in a random direction
    (kept inside the 0.8-scaled workspace and at normalised clearance > `clearance` from the goals already
    placed): neighbourhood moves that still cross each other, instead of workspace-wide crossings."""
    a_w = max(5.0, 1.25 * math.sqrt(n))
    b_w = 3.0
    center = np.array([0.0, 0.0, 1.0])
    rng = np.random.default_rng(seed)
    starts = _draw_points(rng, n, a, b, a_w, b_w, center, clearance)
    goals = []
    for s in starts:
        while True:
            u = rng.normal(size=3)
            u[2] *= b_w / a_w
            p = s + travel * u / np.linalg.norm(u)
            d = p - center
            if (d[0] ** 2 + d[1] ** 2) / (0.8 * a_w) ** 2 + d[2] ** 2 / (0.8 * b_w) ** 2 > 1.0:
                continue
            if all(math.sqrt(((p - q)[0] ** 2 + (p - q)[1] ** 2) / a ** 2 + (p - q)[2] ** 2 / b ** 2) > clearance
                   for q in goals):
                goals.append(p)
                break
    return {
        "n": n, "H": horizon, "T": 0.1 * horizon, "a": a, "b": b,
        "workspace": {"center": center.tolist(), "a_w": a_w, "b_w": b_w},
        "boundary": [{"start": {"p": [float(x) for x in s]}, "goal": {"p": [float(x) for x in g]}}
                     for s, g in zip(starts, goals)],
    }


def random_swarm(n: int, horizon: int, seed: int, **kw):
    return load_problem(random_swarm_doc(n, horizon, seed, **kw))


def config_doc(config: int) -> dict:
    """Reference-schema problem dict of BASELINE config 1..4.

    1 = crossing4 (the reference's scenario); 2 = a 16-robot swarm with workspace-wide random start and goal
    sets (seed 2); 3 and 4 = 32 / 64 robots moving 1.5 m from their starts in random directions (seeds 0 / 2).
    With workspace-wide crossings, 32- and 64-robot swarms almost never reach tol 1e-3 within 500
    iterations under the reference's rho = 1 iteration (0.4% at 32 robots); the neighbourhood moves keep
    the O(n^2) pair interactions and converge for about half of the 32-robot samples
    (tools/scenario_search.py)."""
    if config == 1:
        return CROSSING4
    if config == 2:
        return random_swarm_doc(16, 100, seed=2)
    n, H, seed = {3: (32, 100, 0), 4: (64, 150, 2)}[config]
    return local_swarm_doc(n, H, seed=seed, travel=1.5)


def config_problem(config: int):
    """Problem for BASELINE config 1..4 (1 = crossing4; 2..4 seeded random swarms)."""
    return load_problem(config_doc(config))
