"""(box) Config 3 (4096 samples) with the cooperative careful path on / off (SGSF_NO_COOP)."""
import os, sys, torch
sys.path.insert(0, '.')
import bench
from paper_2501_19042_b200 import SafetyFilter, SolverConfig
prob, shard, B = bench.workload(3, 0, 1, None)
cfg = SolverConfig(max_iters=500, svars=False)
sf = SafetyFilter(prob, degree=10, config=cfg)
xb = torch.from_numpy(shard).cuda()
for no in ("0", "1", "0", "1"):
    os.environ["SGSF_NO_COOP"] = no
    sf.solve_batched(xb, config=cfg); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); out = sf.solve_batched(xb, config=cfg); b.record(); b.synchronize()
    print("no_coop", no, "%.1f ms" % a.elapsed_time(b), int(out.iterations.sum()), int(out.feasible.sum()))
