"""Report whole-batch parity against the real reference's frozen outputs (GPU box).

    python tools/batch_parity.py [batch_cfg2|batch_ws_tight|batch_fuzz ...] [--precision lean strict]

Writes gpurun_out/batch_parity_<name>_<precision>.json (see tests/batch_parity.py for the
classification of iteration-count and verdict flips).
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from tests.batch_parity import compare, run, run_fuzz  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*", default=["batch_cfg2", "batch_ws_tight"])
    ap.add_argument("--precision", nargs="*", default=["strict", "hybrid", "lean"])
    ap.add_argument("--band", type=float, default=1e-6)
    a = ap.parse_args()
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    for name in a.names:
        for prec in a.precision:
            t0 = time.perf_counter()
            g, o = run_fuzz(prec, name) if name.startswith("batch_fuzz") else run(name, prec)
            rep = compare(g, o, a.band)
            rep.update(name=name, precision=prec, band=a.band, wall_s=time.perf_counter() - t0)
            (ROOT / "gpurun_out" / f"batch_parity_{name}_{prec}.json").write_text(json.dumps(rep, indent=1))
            short = {k: v for k, v in rep.items() if not isinstance(v, list)}
            print(json.dumps(short), flush=True)


if __name__ == "__main__":
    main()
