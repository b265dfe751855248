"""(box) Per-sample error of the fused decoder kernel against the module (TF32 off), for a batch > #SMs."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2501_19042_b200 import SafetyFilter, SolverConfig  # noqa: E402
from paper_2501_19042_b200.generative import FusedDecoder, calibrate_batchnorm, make_decoder  # noqa: E402
from paper_2501_19042_b200.initnet import context_features  # noqa: E402
from paper_2501_19042_b200.scenarios import config_problem  # noqa: E402

cfg, kind, B = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
prob = config_problem(cfg)
sf = SafetyFilter(prob, config=SolverConfig(max_iters=50, svars=False))
torch.manual_seed(11)
dec = calibrate_batchnorm(sf, make_decoder(kind, prob.n).cuda())
lat = dec.sample_latent(B, torch.Generator(device="cuda").manual_seed(4), "cuda")
state = torch.as_tensor(context_features(prob), dtype=torch.float32, device="cuda").expand(B, -1, -1)
torch.backends.cuda.matmul.allow_tf32 = False
with torch.no_grad(), torch.backends.cudnn.flags(enabled=True, allow_tf32=False):
    ref = dec(lat, state).double()
f = FusedDecoder(dec)
got = f(lat, state)
torch.cuda.synchronize()
import copy
d64 = copy.deepcopy(dec).double().cpu()
with torch.no_grad():
    ref64 = d64(lat.double().cpu() if kind == "cvae" else lat.cpu(), state.double().cpu()).double().cuda()
print("fp64-vs-torchgpu", float((ref - ref64).abs().max()), "fp64-vs-fused", float((got - ref64).abs().max()))
err = (got - ref).abs().amax(dim=1)
print("scale", float(ref.abs().max()), "max err", float(err.max()), "argmax sample", int(err.argmax()),
      "samples with err > 1e-5:", (err > 1e-5).nonzero().flatten().tolist()[:20])
import time
for _ in range(3):
    f(lat, state)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    f(lat, state)
torch.cuda.synchronize()
print("fused ms", (time.perf_counter() - t0) / 10 * 1e3)
with torch.no_grad():
    for _ in range(3):
        dec(lat, state)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        dec(lat, state)
    torch.cuda.synchronize()
print("torch ms", (time.perf_counter() - t0) / 10 * 1e3)
