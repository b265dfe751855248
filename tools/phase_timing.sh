#!/bin/bash
# (on the GPU box) rebuild with -DSGSF_PHASE_TIMING; per-CTA slot-0 phase cycles -> gpurun_out/pt_*.log
make -C paper_2501_19042_b200/csrc clean >/dev/null
make -C paper_2501_19042_b200/csrc -j16 EXTRA="-DSGSF_PHASE_TIMING ${PT_EXTRA}" >/dev/null 2>&1 || exit 1
mkdir -p gpurun_out
python - <<'PY'
import sys, os
from dataclasses import replace
sys.path.insert(0, ".")
import torch, bench
from paper_2501_19042_b200 import SafetyFilter
def run(tag, x, c, spb=0):
    sys.stdout.flush()
    fd = os.open(f"gpurun_out/pt_{tag}.log", os.O_WRONLY | os.O_CREAT | os.O_TRUNC)
    saved = os.dup(1); os.dup2(fd, 1)
    sf.solve_batched(x, config=c, slots_per_block=spb); torch.cuda.synchronize()
    sys.stdout.flush(); os.dup2(saved, 1); os.close(fd)
import os
if os.environ.get("PT_CONFIG", "2") != "2":
    from paper_2501_19042_b200 import SolverConfig, sample_proposals
    from paper_2501_19042_b200.scenarios import config_problem
    c = int(os.environ["PT_CONFIG"])
    prob = config_problem(c)
    cfg = SolverConfig(max_iters=100 if c == 1 else 500, svars=False)
    sf = SafetyFilter(prob, degree=10, config=cfg)
    xb = torch.from_numpy(sample_proposals(prob, sf.basis, {1: 8, 3: 4096, 4: 8192}[c], seed=0).proposals).cuda()
    run("full", xb, cfg)
    raise SystemExit
prob, shard, cfg = bench.config2_case()
cfg = replace(cfg, precision=os.environ.get("PT_PRECISION", cfg.precision))
sf = SafetyFilter(prob, degree=10, config=cfg)
xb = torch.from_numpy(shard).cuda()
sms = torch.cuda.get_device_properties(0).multi_processor_count
c200 = replace(cfg, max_iters=200, early_stop=False)
run("fixed1", xb[:sms], c200, 1)
run("fixed3", xb[:3 * sms], c200, 3)
run("full", xb, cfg)
PY
