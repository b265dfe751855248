"""(box) Time the config-2 solve per precision in several orders (device-timed), to check independence."""
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_19042_b200 import SafetyFilter  # noqa: E402

prob, shard, cfg = bench.config2_case()
sf = SafetyFilter(prob, degree=10, config=cfg)
xb = torch.from_numpy(shard).cuda()
for prec in sys.argv[1:] or ["lean", "hybrid", "lean", "strict", "lean", "hybrid"]:
    c = replace(cfg, precision=prec)
    sf.solve_batched(xb, config=c)
    ms = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        sf.solve_batched(xb, config=c)
        b.record()
        b.synchronize()
        ms.append(a.elapsed_time(b))
    print(prec, ["%.2f" % m for m in ms], flush=True)
