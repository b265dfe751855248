"""(box) Probe K4's operand layouts with delta inputs and known random weights (identity activation)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2501_19042_b200 import native  # noqa: E402
from paper_2501_19042_b200.generative import _tf32_split  # noqa: E402

torch.manual_seed(0)
L, c0 = 100, 32
c0p = 32
# weights in conv form W[l][o][c][tap]; layer 0 random, layers 1..3 identity at tap 1 (so dbg[0] shows layer 0)
Wl = [torch.randn(128, c0p, 3) * 0.1] + [torch.zeros(128, 128, 3) for _ in range(3)]
for l in range(1, 4):
    Wl[l][:, :, 1] = torch.eye(128)
stages = []
for l, W in enumerate(Wl):
    cinp = W.shape[1]
    for tap in range(3):
        for cg in range(cinp // 32):
            blk = W[:, cg * 32:(cg + 1) * 32, tap].reshape(128, 8, 4).permute(1, 0, 2)
            hi, lo = _tf32_split(blk.float())
            stages.append(torch.cat([hi.reshape(-1), lo.reshape(-1)]))
wpack = torch.cat(stages).cuda()
assert wpack.numel() * 4 == native.load().sgsf_decoder_pack_bytes(c0)
bias = torch.zeros(4 * 128).cuda()
hw, hb = torch.zeros(3 * 128).cuda(), torch.zeros(3).cuda()
ew, eb = torch.zeros(16 * L).cuda(), torch.zeros(16).cuda()
desc = native.Decoder(L, c0, 16, 1, 1.0, 1.0, wpack.data_ptr(), bias.data_ptr(), hw.data_ptr(), hb.data_ptr(),
                      ew.data_ptr(), eb.data_ptr())
probes = [(3, t) for t in list(range(0, 40)) + list(range(60, 100, 3))]
B = len(probes)
h0 = torch.zeros(B, c0, L)
for s, (c, t) in enumerate(probes):
    h0[s, c, t] = 1.0001234
h0 = h0.cuda()
dbg = torch.zeros(B, 4, 128, L, device="cuda")
out = torch.empty(B, 48, dtype=torch.float64, device="cuda")
native.check(native.load().sgsf_decoder_forward_dbg(native.C.byref(desc), B, h0.data_ptr(), out.data_ptr(),
                                                    dbg.data_ptr(), 1, 0), "dbg")
torch.cuda.synchronize()
W0 = Wl[0]
# raw accumulators: P_k[:, r] should be W_k[:, c] at r = t + 1 (the input row), zero elsewhere
for k in range(3):
    bad = []
    for s_, (c, t) in enumerate(probes):
        P = dbg[s_, 1 + k].cpu()
        r = t + 1
        if r < L:
            e = float((P[:, r] - 1.0001234 * W0[:, c, k]).abs().max())
            other = float(P.abs().sum() - P[:, r].abs().sum())
            if e > 1e-5 or other > 1e-4:
                bad.append((r, round(e, 3), round(other, 3)))
    print("P", k, "bad (row, err at row, mass elsewhere):", bad[:4], "...", len(bad))
    errs = []
    for s_, (c, t) in enumerate(probes):
        P = dbg[s_, 1 + k].cpu().double()
        if t + 1 < L:
            errs.append(float(((P[:, t + 1] - 1.0001234 * W0[:, c, k].double()).abs() / W0[:, c, k].double().abs().clamp_min(1e-3)).max()))
    print("   max relative error of the products:", max(errs))
    if bad:
        s_ = [i for i, (c, t) in enumerate(probes) if t + 1 == bad[0][0]][0]
        c = probes[s_][0]
        P = dbg[s_, 1 + k].cpu()[:, bad[0][0]]
        for kk in range(3):
            for cc in range(W0.shape[1]):
                if float((P - W0[:, cc, kk]).abs().max()) < 1e-4:
                    print("     row", bad[0][0], "holds W_%d[:, %d]" % (kk, cc))
        badl = ((P - W0[:, c, k]).abs() > 1e-5).nonzero().flatten().tolist()
        print("     bad lanes:", badl[:40], len(badl))
        print("     their values vs W_k:", [(round(float(P[i]), 4), round(float(W0[i, c, k]), 4)) for i in badl[:6]])
