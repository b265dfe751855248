"""Run the config-2 solve a few times (for ncu / compute-sanitizer captures)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2501_19042_b200 import SafetyFilter, SolverConfig, sample_proposals
from paper_2501_19042_b200.scenarios import config_problem

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=1000)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--max-iters", type=int, default=500)
ap.add_argument("--precision", default="lean")
ap.add_argument("--config", type=int, default=2)
a = ap.parse_args()
prob = config_problem(a.config)
cfg = SolverConfig(max_iters=a.max_iters, svars=False, precision=a.precision)
sf = SafetyFilter(prob, degree=10, config=cfg)
xb = torch.from_numpy(sample_proposals(prob, sf.basis, a.batch, seed=0).proposals).cuda()
for _ in range(a.reps):
    out = sf.solve_batched(xb, config=cfg)
torch.cuda.synchronize()
print("iterations mean", out.iterations.double().mean().item(), "feasible", int(out.feasible.sum().item()))
