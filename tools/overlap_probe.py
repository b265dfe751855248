"""(box) Back-to-back config-2 batches: one stream (each batch's tail idles SMs) against two alternating
streams (the next batch's CTAs start on the SMs the previous batch's tail frees)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_19042_b200 import SafetyFilter  # noqa: E402

prob, shard, cfg = bench.config2_case()
sf = SafetyFilter(prob, degree=10, config=cfg)
xb = torch.from_numpy(shard).cuda()
K = 20
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
for _ in range(3):
    sf.solve_batched(xb, config=cfg)
torch.cuda.synchronize()
for mode in ("1 stream", "2 streams", "1 stream", "2 streams"):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    a.record(cur)
    outs = []
    for k in range(K):
        s = streams[k % 2] if mode == "2 streams" else cur
        s.wait_event(a)
        with torch.cuda.stream(s):
            outs.append(sf.solve_batched(xb, config=cfg).feasible)
    for s in streams:
        cur.wait_stream(s)
    b.record(cur)
    b.synchronize()
    ms = a.elapsed_time(b)
    feas = sum(int(f.sum()) for f in outs)
    print(f"{mode}: {ms / K:.3f} ms per batch, {feas / (ms * 1e-3):.0f} feasible/s")
