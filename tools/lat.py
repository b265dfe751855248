"""Per-iteration latency of one slot vs slots per SM (fixed iteration count, no early stop)."""
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench
from paper_2501_19042_b200 import SafetyFilter

prob, shard, cfg = bench.config2_case()
sf = SafetyFilter(prob, degree=10, config=cfg)
its = 200
cfg2 = replace(cfg, max_iters=its, early_stop=False)
xb = torch.from_numpy(shard).cuda()
sms = torch.cuda.get_device_properties(0).multi_processor_count
for spb in (1, 2, 3):
    B = sms * spb
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for rep in range(3):
        sf.solve_batched(xb[:B], config=cfg2, slots_per_block=spb, timing=ev)
        torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1])
    cyc = ms * 1e-3 * 1.965e9 / its
    print(f"slots/SM {spb}: batch {B}  kernel {ms:.3f} ms  -> {1e3 * ms / its:.2f} us/iter  ({cyc:.0f} cycles/iter), "
          f"SM throughput {spb / cyc * 1e3:.3f} SI per kcycle")
