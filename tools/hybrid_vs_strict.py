"""(box) Random scenarios with early stop: hybrid's iteration counts and verdicts against strict's (FP64
everywhere, which matches the reference on every frozen batch).  A count that differs is listed with strict's
own exit residual at the split, relative to tol (a hybrid FP64 re-evaluation should leave only residuals within
~1e-12 of tol).

    python tools/hybrid_vs_strict.py [scenarios] [seed]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2501_19042_b200 import SafetyFilter, SolverConfig, load_problem, sample_proposals  # noqa: E402
from paper_2501_19042_b200.scenarios import random_swarm_doc  # noqa: E402


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    tot = flips = vflips = 0
    for c in range(cases):
        n = int(rng.choice([3, 4, 6, 8, 12, 16, 24, 32]))
        H = int(rng.choice([30, 50, 100]))
        seed = int(rng.integers(0, 10000))
        spread = float(rng.choice([0.25, 0.6, 1.0]))
        doc = random_swarm_doc(n, H, seed)
        prob = load_problem(doc)
        outs = {}
        for prec in ("strict", "hybrid"):
            cfg = SolverConfig(max_iters=300, svars=False, precision=prec)
            sf = SafetyFilter(prob, degree=10, config=cfg)
            x = torch.from_numpy(sample_proposals(prob, sf.basis, 64, seed=seed, spread=spread).proposals).cuda()
            try:
                outs[prec] = sf.solve_batched(x, config=cfg)
            except NotImplementedError as e:
                outs = None
                print(f"case {c:2d} n={n:2d} H={H:3d}: skipped ({e})")
                break
        if outs is None:
            continue
        a, b = outs["strict"], outs["hybrid"]
        ia, ib = a.iterations.cpu().numpy(), b.iterations.cpu().numpy()
        fa, fb = a.feasible.cpu().numpy(), b.feasible.cpu().numpy()
        hr = a.residual_inf.cpu().numpy()
        bad = np.nonzero(ia != ib)[0]
        detail = []
        for s in bad:
            k = min(ia[s], ib[s]) - 1
            detail.append((int(s), int(ia[s]), int(ib[s]), float(abs(hr[s, k] - 1e-3) / 1e-3)))
        vb = int(((fa != fb) & (ia == ib)).sum())
        tot += len(ia)
        flips += len(bad)
        vflips += vb
        print(f"case {c:2d} n={n:2d} H={H:3d} spread={spread:4.2f}: counts {len(ia) - len(bad)}/{len(ia)} equal, "
              f"verdict flips {vb}" + (f"; flips (sample, strict, hybrid, |res - tol| / tol) {detail}" if detail else ""),
              flush=True)
    print(f"total: {tot - flips}/{tot} counts equal, {vflips} verdict flips at equal counts")


if __name__ == "__main__":
    main()
