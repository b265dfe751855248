"""(box) solve_pipelined with the outputs kept alive vs dropped (keep=False): per-batch time."""
import sys, torch
sys.path.insert(0, '.')
import bench
from paper_2501_19042_b200 import SafetyFilter, SolverConfig
prob, shard, _ = bench.config2_case()
cfg = SolverConfig(max_iters=500, svars=False, precision="hybrid")
sf = SafetyFilter(prob, degree=10, config=cfg)
xb = torch.from_numpy(shard).cuda()
ring = [xb] + [xb.clone() for _ in range(63)]
for keep in (True, False, True, False):
    sf.solve_pipelined((ring[k % 64] for k in range(20)), config=cfg, keep=keep)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    o = sf.solve_pipelined((ring[k % 64] for k in range(20)), config=cfg, keep=keep)
    b.record(); b.synchronize()
    print("keep", keep, "%.3f ms per batch" % (a.elapsed_time(b) / 20))
    del o
