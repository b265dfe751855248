"""Summarise gpurun_out/pt_*.log from tools/phase_timing.sh."""
import re
import sys

import numpy as np

for tag in sys.argv[1:] or ["fixed1", "fixed3", "full"]:
    rows = []
    for ln in open(f"gpurun_out/pt_{tag}.log"):
        if ln.startswith("PT block"):
            rows.append({k: float(v) for k, v in re.findall(r"([A-Za-z0-9]+) ([0-9.]+)", ln)})
    tot = np.array([r["total"] for r in rows])
    its = np.array([r["iters"] for r in rows])
    per = tot / its
    o = np.argsort(-tot)
    print(tag, "CTAs", len(rows), "slot-0 cycles: max %.3g median %.3g" % (tot.max(), np.median(tot)),
          "| cycles/iter median %.0f max %.0f" % (np.median(per), per.max()))
    keys = [k for k in ["T1", "T2", "T3bar", "dec", "G", "MX", "mxG", "mxU", "mxM", "mxP", "mxX", "mxC", "mxE", "t1tc", "t1pos", "t1quiet", "t1ws"] if k in rows[0]]
    for lab, idx in [("slowest", o[:3]), ("median", o[len(o) // 2 - 1:len(o) // 2 + 2])]:
        print("   ", lab, {k: int(np.mean([rows[i][k] for i in idx])) for k in keys}, "iters", [int(its[i]) for i in idx])
