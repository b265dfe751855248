"""(box) 32 robots at the longest two-lane horizon (H = 127): hybrid and lean fit one CTA and solve."""
import sys, torch
sys.path.insert(0, '.')
from paper_2501_19042_b200 import SafetyFilter, SolverConfig, load_problem, sample_proposals
from paper_2501_19042_b200.scenarios import random_swarm_doc
prob = load_problem(random_swarm_doc(32, 127, 3))
for prec in ("hybrid", "lean"):
    cfg = SolverConfig(max_iters=100, svars=False, precision=prec)
    sf = SafetyFilter(prob, degree=10, config=cfg)
    x = torch.from_numpy(sample_proposals(prob, sf.basis, 16, seed=1).proposals).cuda()
    out = sf.solve_batched(x, config=cfg); torch.cuda.synchronize()
    print(prec, "ok", out.iterations.tolist()[:6], int(out.status.sum()))
