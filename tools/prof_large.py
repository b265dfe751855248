"""(box) A short config-4 K1L run for ncu: python tools/prof_large.py [precision [batch [max_iters [early]]]]
(default strict, 256 samples, 60 iterations, no early stop)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_19042_b200 import SafetyFilter, SolverConfig  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "strict"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 60
early = len(sys.argv) > 4 and sys.argv[4] == "1"
prob, shard, B = bench.workload(4, 0, 1, batch)
cfg = SolverConfig(max_iters=iters, early_stop=early, svars=False, precision=prec)
sf = SafetyFilter(prob, degree=10, config=cfg)
xb = torch.from_numpy(shard).cuda()
for _ in range(2):
    out = sf.solve_batched(xb, config=cfg)
torch.cuda.synchronize()
print("ok", float(out.iterations.double().mean()))
