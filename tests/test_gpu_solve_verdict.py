"""The feasible verdict requested through sgsf_solve's outputs (one call: solve, then the verdict kernel
on the same stream) equals a separate sgsf_verdict call on the returned coefficients, bit for bit: ok,
feasible, both margins and both violation counts, for every solve-kernel family (n = 4, 16 with
tensor-core positions, 32 with two lanes per step, strict and lean, and K1L at n = 40)."""
import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _verdict_tensors(B, dev):
    return {"ok": torch.zeros(B, dtype=torch.uint8, device=dev), "feasible": torch.zeros(B, dtype=torch.uint8, device=dev),
            "pmin": torch.zeros(B, dtype=torch.float64, device=dev), "wmax": torch.zeros(B, dtype=torch.float64, device=dev),
            "pc": torch.zeros(B, dtype=torch.int32, device=dev), "wc": torch.zeros(B, dtype=torch.int32, device=dev)}


def _struct(native, t):
    return native.Verdict(t["ok"].data_ptr(), t["feasible"].data_ptr(), t["pmin"].data_ptr(), t["wmax"].data_ptr(),
                          t["pc"].data_ptr(), t["wc"].data_ptr())


@pytest.mark.parametrize("n,horizon,precision", [(4, 50, "lean"), (16, 100, "lean"), (16, 40, "strict"),
                                                 (32, 100, "lean"), (40, 20, "lean")])
def test_fused_verdict_equals_standalone(n, horizon, precision):
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, native, sample_proposals
    from paper_2501_19042_b200.problem import load_problem
    from paper_2501_19042_b200.scenarios import random_swarm_doc
    prob = load_problem(random_swarm_doc(n, horizon, 4))
    cfg = SolverConfig(max_iters=60, svars=False, precision=precision)
    sf = SafetyFilter(prob, config=cfg)
    B = 37
    xb = torch.from_numpy(sample_proposals(prob, sf.basis, B, seed=4, spread=0.6).proposals).cuda()
    dev = xb.device
    lib = native.load()
    handle = sf.operator.handle(cfg.rho, dev)
    dim = sf.coeff_dim
    f64 = dict(dtype=torch.float64, device=dev)
    outs = {k: torch.empty((B, dim), **f64) for k in ("c", "m")}
    hist = {k: torch.empty((B, 60), **f64) for k in ("i", "l")}
    its = torch.empty(B, dtype=torch.int32, device=dev)
    conv = torch.empty(B, dtype=torch.uint8, device=dev)
    disp = torch.empty(B, **f64)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    eqe = torch.empty(B, **f64)
    fused = _verdict_tensors(B, dev)
    vf = _struct(native, fused)
    o = native.Outputs(outs["c"].data_ptr(), outs["m"].data_ptr(), hist["i"].data_ptr(), hist["l"].data_ptr(),
                       its.data_ptr(), conv.data_ptr(), disp.data_ptr(), status.data_ptr(), eqe.data_ptr(), None,
                       C.addressof(vf))
    ccfg = native.Config(60, 1e-3, 1e-8, 1, 1 if precision == "strict" else 0, 0, 0, 0, 1e-3)
    ws = torch.empty(int(lib.sgsf_workspace_bytes(B)), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream().cuda_stream
    native.check(lib.sgsf_solve(handle, B, xb.data_ptr(), None, None, None, C.byref(ccfg), C.byref(o), ws.data_ptr(),
                                None, stream), "sgsf_solve")
    alone = _verdict_tensors(B, dev)
    va = _struct(native, alone)
    native.check(lib.sgsf_verdict(handle, B, outs["c"].data_ptr(), conv.data_ptr(), 1e-3, C.byref(va), stream),
                 "sgsf_verdict")
    torch.cuda.synchronize()
    for k in fused:
        assert torch.equal(fused[k], alone[k]), k
    assert 0 < int(fused["feasible"].sum()) or int(fused["pc"].sum()) > 0   # a non-trivial case
