"""(box) FP64 at 32 robots, H = 100 (config 3's shape): K1 does not fit, K1L takes it.  Its counts and
verdicts against hybrid's on the config-3 batch head, and the time per 512 samples."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_19042_b200 import SafetyFilter, SolverConfig  # noqa: E402

prob, shard, _ = bench.workload(3, 0, 8, None)
xb = torch.from_numpy(shard).cuda()
outs = {}
for prec in ("strict", "hybrid"):
    cfg = SolverConfig(max_iters=500, svars=False, precision=prec)
    sf = SafetyFilter(prob, degree=10, config=cfg)
    sf.solve_batched(xb[:8], config=cfg)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    outs[prec] = sf.solve_batched(xb, config=cfg)
    b.record()
    b.synchronize()
    print(prec, f"{a.elapsed_time(b):.1f} ms for {xb.shape[0]} samples", flush=True)
s, h = outs["strict"], outs["hybrid"]
print("counts equal", int((s.iterations == h.iterations).sum()), "/", s.iterations.numel(),
      "verdicts equal", int((s.feasible == h.feasible).sum()),
      "coeff rel err", float((s.coeffs - h.coeffs).abs().max() / s.coeffs.abs().max()))
