"""How far does the lean (FP32-term) TRAJECTORY move the exit residual, as opposed to its FP32 measurement?

For each config-2 bench sample: solve (want_prev) in the given precision, re-evaluate the exit residual of
the returned iteration in FP64 from the returned iterates (r = F C_k - e(C_{k-1}), the reference's formula
solver.py:330-342 on oracle arithmetic) and compare with the reference's frozen res_inf at that iteration.
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import sf_oracle  # noqa: E402
from tests.batch_parity import proposals  # noqa: E402
from tests.conftest import load_golden  # noqa: E402


def exit_residual(op, Cprev, C):
    pos0 = sf_oracle.positions(op, Cprev)
    d0 = sf_oracle.pair_diffs(op, pos0)
    rel0 = pos0 - op.center[:, None, None]
    *_, tx, ty, tz = sf_oracle.spherical_project(d0[0].ravel(), d0[1].ravel(), d0[2].ravel(), op.lat, op.vert, 1.0, np.inf)
    *_, wx, wy, wz = sf_oracle.spherical_project(rel0[0].ravel(), rel0[1].ravel(), rel0[2].ravel(), op.ws_lat, op.ws_vert, 0.0, 1.0)
    pt = np.stack([tx, ty, tz]).reshape(d0.shape)
    wt = np.stack([wx, wy, wz]).reshape(rel0.shape)
    pos = sf_oracle.positions(op, C)
    rp = sf_oracle.pair_diffs(op, pos) - pt
    rw = (pos - op.center[:, None, None]) - wt
    return max(np.abs(rp).max(), np.abs(rw).max())


def main(precision="lean", limit=1000):
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, load_problem
    g = load_golden("batch_cfg2")
    meta = g["meta"]
    x = proposals("batch_cfg2", meta)[:limit]
    cfg = SolverConfig(precision=precision, svars=False, **meta["config"])
    sf = SafetyFilter(load_problem(meta["problem"]), degree=10, config=cfg)
    out = sf.solve_batched(torch.from_numpy(x).cuda(), config=cfg, want_prev=True)
    torch.cuda.synchronize()
    C, Cp = out.coeffs.cpu().numpy(), out.coeffs_prev.cpu().numpy()
    its = out.iterations.cpu().numpy()
    rinf = out.residual_inf.cpu().numpy()
    op = sf_oracle.make_problem(meta["problem"], degree=10)
    rows = []
    for s in range(len(x)):
        k = int(its[s])
        if k != g["iterations"][s] or k < 2:
            continue
        r64 = exit_residual(op, Cp[s].reshape(3, op.n, op.m1), C[s].reshape(3, op.n, op.m1))
        ref = g["res_inf"][s, k - 1]
        rows.append((s, k, ref, r64, rinf[s, k - 1]))
    a = np.array(rows)
    traj = np.abs(a[:, 3] - a[:, 2]) / a[:, 2]
    meas = np.abs(a[:, 4] - a[:, 3]) / a[:, 3]
    rep = {"precision": precision, "samples": len(rows),
           "trajectory_rel_err": {"median": float(np.median(traj)), "p99": float(np.quantile(traj, 0.99)), "max": float(traj.max())},
           "measurement_rel_err": {"median": float(np.median(meas)), "p99": float(np.quantile(meas, 0.99)), "max": float(meas.max())}}
    print(json.dumps(rep))
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / f"traj_probe_{precision}.json").write_text(json.dumps(rep, indent=1))


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["lean"]), *(int(v) for v in sys.argv[2:3]))
