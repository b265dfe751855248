"""Dump per-sample iteration counts of the benchmark batch (for scheduling analysis)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_2501_19042_b200 import SafetyFilter

prob, shard, cfg = bench.config2_case()
sf = SafetyFilter(prob, degree=10, config=cfg)
out = sf.solve_batched(torch.from_numpy(shard).cuda(), config=cfg)
torch.cuda.synchronize()
Path("gpurun_out").mkdir(exist_ok=True)
np.savez("gpurun_out/iters.npz", iterations=out.iterations.cpu().numpy(), feasible=out.feasible.cpu().numpy(),
         converged=out.converged.cpu().numpy())
print("done", out.iterations.double().mean().item())
