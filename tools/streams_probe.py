"""(box) config-2 batches per ms with 1..4 batches in flight (SafetyFilter.solve_pipelined streams=)."""
import sys, torch
sys.path.insert(0, '.')
import bench
from paper_2501_19042_b200 import SafetyFilter
prob, shard, cfg = bench.config2_case()
sf = SafetyFilter(prob, degree=10, config=cfg)
xb = torch.from_numpy(shard).cuda()
ring = [xb] + [xb.clone() for _ in range(63)]
for ns in (1, 2, 3, 4, 2, 3):
    sf.solve_pipelined((ring[k % 64] for k in range(6)), config=cfg, streams=ns)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    outs = sf.solve_pipelined((ring[k % 64] for k in range(20)), config=cfg, streams=ns)
    b.record(); b.synchronize()
    print(ns, "streams: %.3f ms per batch" % (a.elapsed_time(b) / 20), cfg.precision)
