"""(box) Longest-first queue order on / off (SGSF_NO_ORDER=1), one batch at a time and two in flight (config 2)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_19042_b200 import SafetyFilter, SolverConfig  # noqa: E402

prob, shard, cfg = bench.config2_case()
cfg = SolverConfig(max_iters=500, svars=False, precision=sys.argv[1] if len(sys.argv) > 1 else "hybrid")
sf = SafetyFilter(prob, degree=10, config=cfg)
xb = torch.from_numpy(shard).cuda()
ring = [xb] + [xb.clone() for _ in range(63)]
for no in ("0", "1", "0", "1"):
    os.environ["SGSF_NO_ORDER"] = no
    for ns in (1, 2):
        sf.solve_pipelined((ring[k % 64] for k in range(4)), config=cfg, streams=ns)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        sf.solve_pipelined((ring[k % 64] for k in range(20)), config=cfg, streams=ns)
        b.record()
        b.synchronize()
        print(f"no_order={no} in flight {ns}: {a.elapsed_time(b) / 20:.3f} ms per batch ({cfg.precision})", flush=True)
