"""Decoder -> QP layer -> SF on the device (configs 1-3 pipeline).  The GPU decoder matches the same
random-init module on the CPU to 1e-4 of its output scale (FP32 convolutions; cuDNN's default TF32 is
turned off for the comparison, the pipeline keeps it), and the device pipeline's SF result equals
solve_batched on the same proposals."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,config", [("cvae", 2), ("vqvae", 1)])
def test_decoder_gpu_matches_cpu_and_pipeline(kind, config):
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig
    from paper_2501_19042_b200.generative import decode_proposals, generate_and_filter, make_decoder
    from paper_2501_19042_b200.scenarios import config_problem
    prob = config_problem(config)
    sf = SafetyFilter(prob, config=SolverConfig(max_iters=100, svars=False))
    from paper_2501_19042_b200.generative import calibrate_batchnorm
    from paper_2501_19042_b200.initnet import context_features
    torch.manual_seed(1)
    dec = calibrate_batchnorm(sf, make_decoder(kind, prob.n))
    lat = dec.sample_latent(16, torch.Generator().manual_seed(5))
    state = torch.as_tensor(context_features(prob), dtype=torch.float32).expand(16, -1, -1)
    with torch.no_grad(), torch.backends.cudnn.flags(enabled=True, allow_tf32=False):
        cpu = dec(lat, state)
        gpu = dec.cuda()(lat.cuda(), state.cuda()).cpu()
    scale = float(cpu.abs().max())
    assert float((gpu - cpu).abs().max()) <= 1e-4 * scale
    assert float(cpu.std(dim=0).mean()) > 0.05 * float(cpu.abs().mean())   # the latent matters
    xb, out = generate_and_filter(sf, dec, 64, seed=2)
    assert xb.is_cuda and out.coeffs.shape == (64, sf.coeff_dim)
    assert (out.status == 0).all() and out.eq_err.max().item() <= 1e-8
    ref = sf.solve_batched(xb)
    assert torch.equal(ref.coeffs, out.coeffs) and torch.equal(ref.iterations, out.iterations)


def test_pipeline_graph_replays_the_eager_pipeline():
    """The CUDA-graph pipeline (config 1 size) gives the eager pipeline's results bit for bit, for the
    captured latent and for a new one copied in."""
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig
    from paper_2501_19042_b200.generative import PipelineGraph, calibrate_batchnorm, decode_proposals, make_decoder
    from paper_2501_19042_b200.scenarios import config_problem
    prob = config_problem(1)
    cfg = SolverConfig(max_iters=100, svars=False)
    sf = SafetyFilter(prob, config=cfg)
    torch.manual_seed(3)
    dec = calibrate_batchnorm(sf, make_decoder("cvae", prob.n).cuda())
    g = PipelineGraph(sf, dec, 8, config=cfg, seed=1)
    for latent in (g.latent.clone(), dec.sample_latent(8, torch.Generator(device="cuda").manual_seed(9), "cuda")):
        xb, out = g.replay(latent)
        with torch.no_grad():
            xe = decode_proposals(sf, dec, latent, g.fused)
        ref = sf.solve_batched(xe, config=cfg)
        torch.cuda.synchronize()
        assert torch.equal(xb, xe)
        assert torch.equal(out.coeffs, ref.coeffs) and torch.equal(out.iterations, ref.iterations)
        assert torch.equal(out.feasible, ref.feasible)


@pytest.mark.parametrize("kind,config,batch", [("cvae", 2, 300), ("vqvae", 3, 40), ("cvae", 1, 8)])
def test_fused_decoder_kernel_matches_the_module(kind, config, batch):
    """K4 (sgsf_decoder_forward: the 4 transposed convolutions on tcgen05 3xTF32, head and expansion fused)
    equals the eval-mode PyTorch module in FP32 (TF32 off) to 1e-4 of the output scale, for the CVAE (L = 100
    and L = 25) and the VQ-VAE, over more samples than SMs (the persistent loop)."""
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig
    from paper_2501_19042_b200.generative import FusedDecoder, calibrate_batchnorm, make_decoder
    from paper_2501_19042_b200.initnet import context_features
    from paper_2501_19042_b200.scenarios import config_problem
    prob = config_problem(config)
    sf = SafetyFilter(prob, config=SolverConfig(max_iters=50, svars=False))
    torch.manual_seed(11)
    dec = calibrate_batchnorm(sf, make_decoder(kind, prob.n).cuda())
    lat = dec.sample_latent(batch, torch.Generator(device="cuda").manual_seed(4), "cuda")
    state = torch.as_tensor(context_features(prob), dtype=torch.float32, device="cuda").expand(batch, -1, -1)
    with torch.no_grad(), torch.backends.cudnn.flags(enabled=True, allow_tf32=False):
        torch.backends.cuda.matmul.allow_tf32 = False
        ref = dec(lat, state).double()
    fused = FusedDecoder(dec)
    got = fused(lat, state)
    torch.cuda.synchronize()
    scale = float(ref.abs().max())
    err = float((got - ref).abs().max())
    assert err <= 1e-4 * scale, (err, scale)
    assert got.shape == ref.shape and torch.isfinite(got).all()


def test_fused_decoder_qp_layer_equals_boundary_projection():
    """With the QP layer fused (decode_proposals(..., fused)), K4 returns boundary_projection(line +
    correction) (projection.py:11-25): equal to the module path to 1e-4 of the scale, endpoint conditions
    to 1e-9."""
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig
    from paper_2501_19042_b200.generative import FusedDecoder, calibrate_batchnorm, decode_proposals, make_decoder
    from paper_2501_19042_b200.scenarios import config_problem
    prob = config_problem(2)
    sf = SafetyFilter(prob, config=SolverConfig(max_iters=50, svars=False))
    torch.manual_seed(2)
    dec = calibrate_batchnorm(sf, make_decoder("cvae", prob.n).cuda())
    lat = dec.sample_latent(200, torch.Generator(device="cuda").manual_seed(8), "cuda")
    with torch.no_grad(), torch.backends.cudnn.flags(enabled=True, allow_tf32=False):
        ref = decode_proposals(sf, dec, lat)
    got = decode_proposals(sf, dec, lat, FusedDecoder(dec))
    torch.cuda.synchronize()
    assert float((got - ref).abs().max()) <= 1e-4 * float(ref.abs().max())
    res = got.cpu().numpy()
    for b in range(0, 200, 37):
        assert abs(sf.equality.residual(res[b])).max() <= 1e-9
