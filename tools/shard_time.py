"""(box) Strong-scaling estimate on one GPU: the device time of rank 0's shard of config 3 / 4 for world sizes
1, 2, 4, 8 (each rank solves its shard with no collective in the solve; the N-GPU step is the max over ranks).
python tools/shard_time.py <config> [precision]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_19042_b200 import SafetyFilter, SolverConfig  # noqa: E402

config = int(sys.argv[1]) if len(sys.argv) > 1 else 3
prec = sys.argv[2] if len(sys.argv) > 2 else "hybrid"
base = None
for world in (1, 2, 4, 8):
    ms_max = 0.0
    for rank in sorted({0, world - 1}):
        prob, shard, B = bench.workload(config, rank, world, None)
        cfg = SolverConfig(max_iters=bench.max_iters_of(config), svars=False, precision=prec)
        sf = SafetyFilter(prob, degree=10, config=cfg)
        xb = torch.from_numpy(shard).cuda()
        sf.solve_batched(xb, config=cfg)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        sf.solve_batched(xb, config=cfg)
        b.record()
        b.synchronize()
        ms_max = max(ms_max, a.elapsed_time(b))
    base = base or ms_max
    print(f"config {config} world {world}: shard {shard.shape[0]} samples, {ms_max:.1f} ms (first/last rank max), "
          f"speed-up {base / ms_max:.2f}x, efficiency {base / ms_max / world:.2f}", flush=True)
