"""Compare GPU solve (lean/strict) with a golden case iteration by iteration."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from tests.conftest import load_golden
from paper_2501_19042_b200 import SafetyFilter, SolverConfig, load_problem

name = sys.argv[1] if len(sys.argv) > 1 else "crossing4_cfg1"
case = load_golden(name)
meta = case["meta"]
prob = load_problem(meta["problem"])
for prec in ("strict", "lean"):
    cfg = SolverConfig(precision=prec, svars=False, **meta["config"])
    sf = SafetyFilter(prob, degree=meta["degree"], config=cfg)
    out = sf.solve_batched(torch.from_numpy(case["proposals"]).cuda(), config=cfg)
    its = out.iterations.cpu().numpy()
    ri = out.residual_inf.cpu().numpy()
    for s in range(min(3, len(its))):
        k = int(min(its[s], case["iterations"][s]))
        rel = np.abs(ri[s, :k] - case["res_inf"][s, :k]) / case["res_inf"][s, :k]
        first = int(np.argmax(rel > 1e-3)) if (rel > 1e-3).any() else -1
        print(prec, s, "its", its[s], case["iterations"][s], "first hist mismatch at", first,
              "ours", ri[s, max(first, 0):max(first, 0) + 3], "ref", case["res_inf"][s, max(first, 0):max(first, 0) + 3])
