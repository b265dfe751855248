"""(box) K1L A/B: digest and kernel time of a config-4 shard and the large fuzz scenarios.

    python tools/k1l_ab.py [batch]      # prints one JSON line: sha256 of (iterations, coeffs) and ms per solve
"""
import hashlib
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_19042_b200 import SafetyFilter, SolverConfig  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
h = hashlib.sha256()
res = {}
for prec in ("hybrid", "strict", "lean"):
    prob, shard, B = bench.workload(4, 0, 1, batch)
    cfg = SolverConfig(max_iters=1000, svars=False, precision=prec)
    sf = SafetyFilter(prob, degree=10, config=cfg)
    xb = torch.from_numpy(shard).cuda()
    out = sf.solve_batched(xb, config=cfg)
    ms = []
    for _ in range(2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        out = sf.solve_batched(xb, config=cfg)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    h.update(out.iterations.cpu().numpy().tobytes())
    h.update(out.coeffs.cpu().numpy().tobytes())
    res[prec] = {"ms": ms, "iters": float(out.iterations.double().mean())}
from tests.batch_parity import run_fuzz  # noqa: E402
for prec in ("hybrid", "strict", "lean"):
    g, o = run_fuzz(prec, "batch_fuzz_large")
    h.update(o["iterations"].tobytes())
    h.update(np.nan_to_num(o["coeffs"]).tobytes())
print(json.dumps({"digest": h.hexdigest(), **res}), flush=True)
