"""(box) BASELINE config 5 across scenarios: the init network trained on 16 random 16-drone scenarios
(H = 100) through the differentiable SF, then every start strategy evaluated on the bench scenario
(config 2) and on 4 scenarios it never saw.  Writes gpurun_out/config5_multi.json.

    python tools/config5_multi.py [--train 16] [--steps 2000] [--iters 20]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2501_19042_b200 import SafetyFilter, SolverConfig, sample_proposals  # noqa: E402
from paper_2501_19042_b200.initnet import InitNet, init_sweep, train_init_net_multi  # noqa: E402
from paper_2501_19042_b200.scenarios import config_problem, random_swarm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--train", type=int, default=16)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--pool", type=int, default=2048)
    a = ap.parse_args()
    torch.manual_seed(0)
    cfg = SolverConfig(max_iters=500)
    train = []
    for s in range(a.train):
        sf = SafetyFilter(random_swarm(16, 100, seed=100 + s), config=cfg)
        pool = torch.from_numpy(sample_proposals(sf.problem, sf.basis, a.pool, seed=1).proposals).cuda()
        train.append((sf, pool))
    net = InitNet(16, train[0][0].coeff_dim)
    log = train_init_net_multi(train, net, iters=a.iters, steps=a.steps)
    evals = {"config2 (seed 2)": config_problem(2)}
    for s in range(4):
        evals[f"unseen seed {200 + s}"] = random_swarm(16, 100, seed=200 + s)
    res = {}
    for name, prob in evals.items():
        sf = SafetyFilter(prob, config=cfg)
        xs = torch.from_numpy(sample_proposals(prob, sf.basis, 1000, seed=0).proposals).cuda()
        r = init_sweep(sf, xs, net, strategies=("projected", "initnet"), max_iters=500, trace_iters=10)
        res[name] = {k: {kk: v[kk] for kk in ("mean_iterations", "converged", "feasible")} for k, v in r.items()}
        print(f"{name:18s} projected {r['projected']['mean_iterations']:6.1f} its / feas {r['projected']['feasible']:.3f}"
              f"   initnet {r['initnet']['mean_iterations']:6.1f} its / feas {r['initnet']['feasible']:.3f}", flush=True)
    out = {"train_scenarios": a.train, "steps": a.steps, "K": a.iters, "training_seconds": log.seconds,
           "sf_seconds": log.sf_seconds, "loss_first": log.losses[:5], "loss_last": log.losses[-5:], "eval": res}
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/config5_multi.json", "w") as fh:
        json.dump(out, fh, indent=1)
    rel = [1 - v["initnet"]["mean_iterations"] / v["projected"]["mean_iterations"] for v in res.values()]
    print(f"training {log.steps} steps in {log.seconds:.1f} s; mean iteration cut {100 * np.mean(rel):.1f}%")


if __name__ == "__main__":
    main()
