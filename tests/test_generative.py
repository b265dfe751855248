"""Generative decoders (configs 1-3 inputs), host side: shapes, seeded sampling, and the QP layer
(decoded proposals meet the start/goal conditions)."""
import numpy as np
import pytest
import torch

from paper_2501_19042_b200 import SafetyFilter
from paper_2501_19042_b200.generative import calibrate_batchnorm, decode_proposals, latent_length, make_decoder
from paper_2501_19042_b200.scenarios import config_problem


@pytest.mark.parametrize("kind,config", [("cvae", 1), ("vqvae", 1), ("cvae", 2)])
def test_decoded_proposals_meet_boundary_conditions(kind, config):
    prob = config_problem(config)
    sf = SafetyFilter(prob)
    torch.manual_seed(0)
    dec = calibrate_batchnorm(sf, make_decoder(kind, prob.n), batches=2, batch=64)
    assert dec.L == latent_length(prob.n) == (25 if prob.n <= 8 else 100)
    g = torch.Generator().manual_seed(3)
    lat = dec.sample_latent(6, g)
    with torch.no_grad():
        xb = decode_proposals(sf, dec, lat)
    assert xb.shape == (6, sf.coeff_dim) and xb.dtype == torch.float64
    res = np.stack([sf.equality.residual(x) for x in xb.numpy()])
    assert np.abs(res).max() <= 1e-9
    with torch.no_grad():
        again = decode_proposals(sf, dec, dec.sample_latent(6, torch.Generator().manual_seed(3)))
    assert torch.equal(xb, again)
    assert float(xb.std(dim=0).max()) > 1e-2   # samples differ


def test_vq_indices_in_codebook():
    dec = make_decoder("vqvae", 16)
    idx = dec.sample_latent(100, torch.Generator().manual_seed(0))
    assert idx.shape == (100, 100) and int(idx.min()) >= 0 and int(idx.max()) < 512
