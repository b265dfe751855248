"""(box) Where the decode + QP time goes in the pipeline: host overhead vs the K4 kernel."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2501_19042_b200 import SafetyFilter, SolverConfig  # noqa: E402
from paper_2501_19042_b200.generative import FusedDecoder, calibrate_batchnorm, decode_proposals, make_decoder  # noqa: E402
from paper_2501_19042_b200.scenarios import config_problem  # noqa: E402

prob = config_problem(2)
sf = SafetyFilter(prob, config=SolverConfig(max_iters=500, svars=False))
torch.manual_seed(0)
dec = calibrate_batchnorm(sf, make_decoder("cvae", prob.n).cuda()).eval()
fused = FusedDecoder(dec)
gen = torch.Generator(device="cuda").manual_seed(0)
lat = dec.sample_latent(1000, gen, "cuda")
for _ in range(3):
    decode_proposals(sf, dec, lat, fused)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for mode in ("pipelined", "single"):
    t0 = time.perf_counter()
    ev[0].record()
    reps = 20 if mode == "pipelined" else 1
    for _ in range(reps):
        xb = decode_proposals(sf, dec, lat, fused)
    ev[1].record()
    t_host = (time.perf_counter() - t0) / reps
    ev[1].synchronize()
    print(mode, "device ms per call %.3f" % (ev[0].elapsed_time(ev[1]) / reps), "host ms per call %.3f" % (t_host * 1e3))
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(20):
    decode_proposals(sf, dec, lat, fused)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(8)
