"""(box) Layer-by-layer comparison of the fused decoder kernel (K4) against an FP64 restatement."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2501_19042_b200 import SafetyFilter, SolverConfig, native  # noqa: E402
from paper_2501_19042_b200.generative import FusedDecoder, calibrate_batchnorm, make_decoder  # noqa: E402
from paper_2501_19042_b200.initnet import context_features  # noqa: E402
from paper_2501_19042_b200.scenarios import config_problem  # noqa: E402

prob = config_problem(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
sf = SafetyFilter(prob, config=SolverConfig(max_iters=50, svars=False))
torch.manual_seed(11)
dec = calibrate_batchnorm(sf, make_decoder("cvae", prob.n).cuda())
B = 3
lat = dec.sample_latent(B, torch.Generator(device="cuda").manual_seed(4), "cuda")
state = torch.as_tensor(context_features(prob), dtype=torch.float32, device="cuda").expand(B, -1, -1)
f = FusedDecoder(dec)
h0 = f.first_layer_input(lat, state)
L = dec.L
dbg = torch.zeros(B, 4, 128, L, device="cuda")
out = torch.empty(B, 3 * f.nm1, dtype=torch.float64, device="cuda")
native.check(native.load().sgsf_decoder_forward_dbg(native.C.byref(f._desc(f.c0, None, None)), B, h0.data_ptr(), out.data_ptr(),
                                                    dbg.data_ptr(), 0, 0), "dbg")
torch.cuda.synchronize()
convs = [m for m in dec.body if isinstance(m, torch.nn.ConvTranspose1d)]
bns = [m for m in dec.body if isinstance(m, torch.nn.modules.batchnorm._BatchNorm)]
import copy
convs = [copy.deepcopy(m).double().cpu() for m in convs]
bns = [copy.deepcopy(m).double().cpu() for m in bns]
x = h0.double().cpu()
for li, (cv, bn) in enumerate(zip(convs, bns)):
    with torch.no_grad():
        y = bn(cv(x)).double()
        y = torch.where(y > 0, y, 0.01 * y).cuda()
    g = dbg[:, li].double()
    print("layer", li, "max|ref|", float(y.abs().max()), "err", float((g - y).abs().max()),
          "err first pos", float((g[..., 0] - y[..., 0]).abs().max()), "err mid", float((g[..., L // 2] - y[..., L // 2]).abs().max()))
    if li == 0:
        # which taps: compare against each single-tap partial
        pass
    x = y.cpu()
with torch.no_grad():
    ref = dec(lat, state).double()
print("out err", float((out - ref).abs().max()), float(ref.abs().max()))
cv, bn = convs[0], bns[0]
Wt = cv.weight.detach().double().cpu()
Wc = Wt.flip(2).permute(1, 0, 2).contiguous()
sc = bn.weight.double().cpu() / torch.sqrt(bn.running_var.double().cpu() + bn.eps)
Wc = Wc * sc[:, None, None]
b0 = (cv.bias.double().cpu() - bn.running_mean.double().cpu()) * sc + bn.bias.double().cpu()
Path("gpurun_out").mkdir(exist_ok=True)
torch.save({"h0": h0.cpu(), "dbg": dbg.cpu(), "W0": Wc, "b0": b0}, "gpurun_out/dec_dbg.pt")
