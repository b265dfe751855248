"""(box) Config-3 shards: kernel time against the iteration counts they contain (strong-scaling diagnosis)."""
import sys, torch
sys.path.insert(0, '.')
import bench
from paper_2501_19042_b200 import SafetyFilter, SolverConfig
for world, rank in ((1, 0), (8, 0), (8, 7)):
    prob, shard, B = bench.workload(3, rank, world, None)
    cfg = SolverConfig(max_iters=500, svars=False)
    sf = SafetyFilter(prob, degree=10, config=cfg)
    xb = torch.from_numpy(shard).cuda()
    sf.solve_batched(xb, config=cfg); torch.cuda.synchronize()
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    out = sf.solve_batched(xb, config=cfg, timing=ev); torch.cuda.synchronize()
    it = out.iterations.double()
    print(world, rank, xb.shape[0], "kernel ms %.1f" % ev[0].elapsed_time(ev[1]), "iters mean %.0f max %.0f" % (it.mean(), it.max()),
          "sum/148 slots %.0f" % (it.sum() / 148))
