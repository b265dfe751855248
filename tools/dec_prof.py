"""(box) Fused decoder + QP launches: python tools/dec_prof.py [config [cvae|vqvae [batch]]] (for ncu -k regex:decoder)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2501_19042_b200 import SafetyFilter, SolverConfig  # noqa: E402
from paper_2501_19042_b200.generative import FusedDecoder, calibrate_batchnorm, decode_proposals, make_decoder  # noqa: E402
from paper_2501_19042_b200.scenarios import config_problem  # noqa: E402

prob = config_problem(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
kind = sys.argv[2] if len(sys.argv) > 2 else "cvae"
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
sf = SafetyFilter(prob, config=SolverConfig(max_iters=50, svars=False))
torch.manual_seed(0)
dec = calibrate_batchnorm(sf, make_decoder(kind, prob.n).cuda()).eval()
fused = FusedDecoder(dec)
lat = dec.sample_latent(B, torch.Generator(device="cuda").manual_seed(0), "cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for _ in range(3):
    decode_proposals(sf, dec, lat, fused)
ev[0].record()
for _ in range(20):
    decode_proposals(sf, dec, lat, fused)
ev[1].record()
ev[1].synchronize()
print("decode+QP ms per batch %.4f" % (ev[0].elapsed_time(ev[1]) / 20))
