"""(box) BASELINE config 5: init network vs zero / heuristic starts, with the differentiable SF backward.

Config-2 problem (16 drones, H=100).  The init net trains on a pool of proposals (seed 1) through
K unrolled SF steps (CUDA forward + reverse kernels).  Every strategy is then evaluated on the bench's
1000 proposals (seed 0) with the device solver (max_iters 500, tol 1e-3).

Also times the unrolled SF alone: forward + backward of K steps for a 1000-sample batch (CUDA events).
Writes gpurun_out/config5.json.

    python tools/config5_sweep.py [--steps 1500] [--iters 20] [--batch 256]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2501_19042_b200 import SafetyFilter, SolverConfig, sample_proposals  # noqa: E402
from paper_2501_19042_b200.initnet import InitNet, init_sweep, train_init_net  # noqa: E402
from paper_2501_19042_b200.scenarios import config_problem  # noqa: E402
from paper_2501_19042_b200.unrolled import fixed_point_loss, unrolled_solve  # noqa: E402


def time_unrolled(sf, xb, iters, reps=5):
    x = xb.clone().requires_grad_(True)
    for _ in range(2):
        fixed_point_loss(unrolled_solve(sf, x, iters=iters), x).backward()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fwd = tot = 0.0
    for _ in range(reps):
        s.record()
        it = unrolled_solve(sf, x, iters=iters)
        e.record()
        e.synchronize()
        fwd += s.elapsed_time(e)
        s.record()
        it = unrolled_solve(sf, x, iters=iters)
        fixed_point_loss(it, x).backward()
        e.record()
        e.synchronize()
        tot += s.elapsed_time(e)
    return fwd / reps, tot / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=1500)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--pool", type=int, default=8192)
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--out", default="gpurun_out/config5.json")
    a = ap.parse_args()
    torch.manual_seed(0)
    prob = config_problem(2)
    sf = SafetyFilter(prob, config=SolverConfig(max_iters=500))
    pool = torch.from_numpy(sample_proposals(prob, sf.basis, a.pool, seed=1).proposals).cuda()
    evalset = torch.from_numpy(sample_proposals(prob, sf.basis, 1000, seed=0).proposals).cuda()

    fwd_ms, fb_ms = time_unrolled(sf, evalset, a.iters)
    net = InitNet(prob.n, sf.coeff_dim)
    t0 = time.perf_counter()
    log = train_init_net(sf, net, pool, iters=a.iters, steps=a.steps, batch=a.batch, lr=a.lr)
    train_s = time.perf_counter() - t0
    res = init_sweep(sf, evalset, net, max_iters=500, trace_iters=100)
    out = {
        "workload": "config 2 problem (16 drones, H=100), 1000 eval proposals (seed 0), "
                    f"init net trained on {a.pool} proposals (seed 1)",
        "unrolled_sf": {"iters": a.iters, "batch": 1000, "forward_ms": fwd_ms, "forward_backward_ms": fb_ms,
                        "sample_steps_per_s_fwd_bwd": 1000 * a.iters / (fb_ms / 1e3)},
        "training": {"steps": log.steps, "batch": a.batch, "K": a.iters, "lr": a.lr, "seconds": train_s,
                     "sf_seconds": log.sf_seconds, "loss_first": log.losses[:5], "loss_last": log.losses[-5:]},
        "strategies": res,
    }
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print(f"unrolled SF K={a.iters} B=1000: forward {fwd_ms:.2f} ms, forward+backward {fb_ms:.2f} ms")
    print(f"training: {log.steps} steps in {train_s:.1f} s (SF {log.sf_seconds:.1f} s); "
          f"loss {sum(log.losses[:5]) / 5:.4g} -> {sum(log.losses[-5:]) / 5:.4g}")
    for s, r in res.items():
        print(f"{s:10s} mean its {r['mean_iterations']:7.1f}  median {r['median_iterations']:6.1f}  "
              f"converged {r['converged']:.3f}  feasible {r['feasible']:.3f}  "
              f"res@10 {r['residual_trace'][9]:.3g}  res@100 {r['residual_trace'][-1]:.3g}")


if __name__ == "__main__":
    main()
