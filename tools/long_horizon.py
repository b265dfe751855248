"""(box) Long horizons that must keep fitting one CTA: n = 4 at H = 300 (hybrid, lean, strict) and n = 32 at
H = 127 (hybrid, lean)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2501_19042_b200 import SafetyFilter, SolverConfig, load_problem, sample_proposals  # noqa: E402
from paper_2501_19042_b200.scenarios import random_swarm_doc  # noqa: E402

for n, H, precs in ((4, 300, ("hybrid", "lean", "strict")), (32, 127, ("hybrid", "lean"))):
    prob = load_problem(random_swarm_doc(n, H, 3))
    for prec in precs:
        cfg = SolverConfig(max_iters=50, svars=False, precision=prec)
        sf = SafetyFilter(prob, degree=10, config=cfg)
        x = torch.from_numpy(sample_proposals(prob, sf.basis, 8, seed=1).proposals).cuda()
        out = sf.solve_batched(x, config=cfg)
        torch.cuda.synchronize()
        print(f"n={n} H={H} {prec}: ok, status {int(out.status.abs().sum())}, iterations {out.iterations.tolist()}")

# 64 robots at H = 170 in FP64: phase B's partials do not fit next to the FP64 state, the launcher falls back
prob = load_problem(random_swarm_doc(64, 170, 5))
for prec in ("strict", "hybrid"):
    cfg = SolverConfig(max_iters=30, svars=False, precision=prec)
    sf = SafetyFilter(prob, degree=10, config=cfg)
    x = torch.from_numpy(sample_proposals(prob, sf.basis, 4, seed=1).proposals).cuda()
    out = sf.solve_batched(x, config=cfg)
    torch.cuda.synchronize()
    print(f"n=64 H=170 {prec}: ok, status {int(out.status.abs().sum())}, iterations {out.iterations.tolist()}")
