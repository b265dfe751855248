"""(box) Search seeded swarm scenarios for BASELINE configs 3/4 whose samples converge within max_iters
(the round-1 config-3 scenario, workspace-wide random start/goal sets, converged for 0.4% within 500).

    python tools/scenario_search.py N H BATCH MAX_ITERS
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2501_19042_b200 import SafetyFilter, SolverConfig, load_problem, sample_proposals  # noqa: E402
from paper_2501_19042_b200.scenarios import local_swarm_doc  # noqa: E402

n, H, batch, mi = (int(v) for v in sys.argv[1:5])
for travel in (1.5, 2.5, 4.0, 6.0):
    for seed in range(3):
        prob = load_problem(local_swarm_doc(n, H, seed, travel))
        cfg = SolverConfig(max_iters=mi, svars=False, precision="lean" if n <= 32 else "strict")
        sf = SafetyFilter(prob, degree=10, config=cfg)
        x = torch.from_numpy(sample_proposals(prob, sf.basis, batch, seed=0).proposals).cuda()
        out = sf.solve_batched(x, config=cfg)
        its = out.iterations.double()
        print(json.dumps({"n": n, "H": H, "seed": seed, "travel": travel,
                          "converged": float(out.converged.double().mean()),
                          "feasible": float(out.feasible.double().mean()), "mean_its": float(its.mean()),
                          "median_its": float(its.median())}), flush=True)
