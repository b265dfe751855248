"""Time the SF on a BASELINE config (device-timed, CUDA events), e.g. `python tools/config_bench.py 3`.

Config 2 is bench.py's workload; this tool reports the other configs' single-GPU numbers for DESIGN.md.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2501_19042_b200 import SafetyFilter, SolverConfig, sample_proposals
from paper_2501_19042_b200.scenarios import config_problem

config = int(sys.argv[1]) if len(sys.argv) > 1 else 3
batch = int(sys.argv[2]) if len(sys.argv) > 2 else {1: 8, 2: 1000, 3: 4096, 4: 8192}[config]
max_iters = 100 if config == 1 else 500
prob = config_problem(config)
cfg = SolverConfig(max_iters=max_iters, svars=False)
sf = SafetyFilter(prob, config=cfg)
xb = torch.from_numpy(sample_proposals(prob, sf.basis, batch, seed=0).proposals).cuda()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for rep in range(3):
    torch.cuda.synchronize()
    ev[0].record()
    out = sf.solve_batched(xb, config=cfg)
    ev[1].record()
    torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1])
its = out.iterations.double()
print(f"config {config}: n={prob.n} H={prob.horizon_samples - 1} batch {batch}: {ms:.2f} ms, "
      f"{int(out.feasible.sum())} feasible ({out.feasible.double().mean().item():.3f}), mean iterations "
      f"{its.mean().item():.1f}, max {int(its.max().item())} -> {1e3 * out.feasible.sum().item() / ms:.0f} feasible/s, "
      f"{its.sum().item() / ms / 1e3:.2f} M sample-iterations/s")
