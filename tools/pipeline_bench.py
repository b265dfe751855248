"""(box) The generative pipeline of BASELINE configs 1-3 on one B200, all on the device:
latent -> decoder (random-init CVAE / VQ-VAE) -> boundary QP layer -> SF kernel -> verdict.
Times each stage with CUDA events (after warm-up) and writes gpurun_out/pipeline.json.

    python tools/pipeline_bench.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2501_19042_b200 import SafetyFilter, SolverConfig  # noqa: E402
from paper_2501_19042_b200.generative import FusedDecoder, calibrate_batchnorm, decode_proposals, make_decoder  # noqa: E402
from paper_2501_19042_b200.scenarios import config_problem  # noqa: E402

CASES = [  # (config, decoder, batch, max_iters)
    (1, "cvae", 8, 100),
    (2, "cvae", 1000, 500),
    (3, "vqvae", 4096, 500),
]


def run(config, kind, batch, max_iters, reps=3):
    torch.manual_seed(0)
    prob = config_problem(config)
    sf = SafetyFilter(prob, config=SolverConfig(max_iters=max_iters, svars=False))
    dec = calibrate_batchnorm(sf, make_decoder(kind, prob.n).cuda())
    fused = FusedDecoder(dec)   # K4
    gen = torch.Generator(device="cuda").manual_seed(0)
    # one warm-up pass (cuDNN plans, allocator blocks), then `reps` passes enqueued back to back: the stage
    # times are the device's, not the host's launch latency after a synchronisation
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(reps + 1)]
    out = None
    t_dec = t_sf = 0.0
    keep = []
    for r in range(reps + 1):
        with torch.no_grad():
            ev[r][0].record()
            xb = decode_proposals(sf, dec, dec.sample_latent(batch, gen, "cuda"), fused)
            ev[r][1].record()
            out = sf.solve_batched(xb)
            ev[r][2].record()
        keep.append((xb, out))
        if r == 0:
            ev[0][2].synchronize()
    ev[reps][2].synchronize()
    for r in range(1, reps + 1):
        t_dec += ev[r][0].elapsed_time(ev[r][1]) / reps
        t_sf += ev[r][1].elapsed_time(ev[r][2]) / reps
    its = out.iterations.double()
    return {"config": config, "decoder": kind, "batch": batch, "n": prob.n, "H": prob.horizon_samples - 1,
            "max_iters": max_iters, "decode_qp_ms": t_dec, "sf_verdict_ms": t_sf, "total_ms": t_dec + t_sf,
            "mean_iterations": float(its.mean()), "converged": float(out.converged.double().mean()),
            "feasible": float(out.feasible.double().mean()),
            "feasible_per_s": float(out.feasible.double().sum()) / ((t_dec + t_sf) / 1e3)}


def main():
    rows = [run(*c) for c in CASES]
    graph = graph_vs_eager()
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/pipeline.json", "w") as fh:
        json.dump({"note": "random-init decoders (no trained weights exist offline); all stages on one B200",
                   "rows": rows, "config1_graph": graph}, fh, indent=1)
    for r in rows:
        print(f"config {r['config']} {r['decoder']:5s} B={r['batch']:5d}: decode+QP {r['decode_qp_ms']:.2f} ms, "
              f"SF+verdict {r['sf_verdict_ms']:.2f} ms, iterations {r['mean_iterations']:.1f}, "
              f"converged {r['converged']:.3f}, feasible {r['feasible']:.3f}")



def graph_vs_eager(reps=20):
    """Config 1 (8 samples, launch-bound): the eager pipeline against its CUDA-graph replay."""
    from paper_2501_19042_b200.generative import PipelineGraph
    prob = config_problem(1)
    cfg = SolverConfig(max_iters=100, svars=False)
    sf = SafetyFilter(prob, config=cfg)
    torch.manual_seed(0)
    dec = calibrate_batchnorm(sf, make_decoder("cvae", prob.n).cuda())
    g = PipelineGraph(sf, dec, 8, config=cfg)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        g.replay()
    s.record()
    for _ in range(reps):
        g.replay()
    e.record()
    e.synchronize()
    graph_ms = s.elapsed_time(e) / reps
    with torch.no_grad():
        for _ in range(3):
            sf.solve_batched(decode_proposals(sf, dec, g.latent), config=cfg)
        s.record()
        for _ in range(reps):
            sf.solve_batched(decode_proposals(sf, dec, g.latent), config=cfg)
        e.record()
        e.synchronize()
    eager_ms = s.elapsed_time(e) / reps
    print(f"config 1 pipeline (decode + QP + SF + verdict, 8 samples): eager {eager_ms:.2f} ms, CUDA graph {graph_ms:.2f} ms")
    return {"eager_ms": eager_ms, "graph_ms": graph_ms}


if __name__ == "__main__":
    main()
