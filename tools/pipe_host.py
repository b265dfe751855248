"""(box) Host-side enqueue time of each config-2 pipeline stage (does any stage block the host?)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2501_19042_b200 import SafetyFilter, SolverConfig
from paper_2501_19042_b200.generative import FusedDecoder, calibrate_batchnorm, decode_proposals, make_decoder
from paper_2501_19042_b200.initnet import FoldedInitNet, InitNet, initial_states
from paper_2501_19042_b200.unrolled import device_constants_of
from paper_2501_19042_b200.scenarios import config_problem
prob = config_problem(2)
torch.manual_seed(0)
sf = SafetyFilter(prob, degree=10, config=SolverConfig(max_iters=500, svars=False))
dec = calibrate_batchnorm(sf, make_decoder("cvae", prob.n).cuda()).eval()
fused = FusedDecoder(dec)
net = FoldedInitNet(InitNet(prob.n, sf.coeff_dim).cuda().eval(), device_constants_of(sf, "cuda")["context"][None])
gen = torch.Generator(device="cuda").manual_seed(0)
for r in range(6):
    t = [time.perf_counter()]
    with torch.no_grad():
        lat = dec.sample_latent(1000, gen, "cuda"); t.append(time.perf_counter())
        xb = decode_proposals(sf, dec, lat, fused); t.append(time.perf_counter())
        xi0, lam0 = initial_states(sf, xb, "initnet", net); t.append(time.perf_counter())
        out = sf.solve_batched(xb, xi0=xi0, lam0=lam0); t.append(time.perf_counter())
    print(["%.3f" % (1e3 * (b - a)) for a, b in zip(t, t[1:])])
torch.cuda.synchronize()
