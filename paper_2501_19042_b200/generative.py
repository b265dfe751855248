"""Generative proposal decoders (CVAE / VQ-VAE) feeding the safety filter on the device.

BASELINE configs 1-3 sample their SF inputs from a CVAE or VQ-VAE decoder. The reference package
has no network. These modules follow the paper's descriptions
(PAPER.md "VQ-VAE Network Details", "CVAE Network Details", :302-307):

* CVAE decoder:
  * a Gaussian latent Z of L x 3;
  * a state network of two convolution layers (ReLU, batch norm) over the per-robot start/goal
    states, concatenated with the latent;
  * 4 transposed-convolution layers with 128 channels, LeakyReLU, batch norm and dropout.
* VQ-VAE decoder:
  * a codebook of 512 three-dimensional vectors and L latent positions;
  * 4 transposed-convolution layers with 128 channels, ReLU, batch norm and dropout.
  * Without a trained PixelCNN prior, the code indices are sampled uniformly.

Both decoders emit a correction xi' to the straight-line coefficients. The differentiable QP layer
of the paper (the boundary projection, ``projection.py:11-25``) turns it into xi_bar, which
:func:`generate_and_filter` hands to the SF kernel without leaving the device.

The weights are random-init (BASELINE config 1: "random-init decoder"); :func:`calibrate_batchnorm`
sets their batch-norm statistics from sampled latents so that the samples differ. The parity target
is the same module on the CPU with the same weights (``tests/test_gpu_generative.py``).
"""
from __future__ import annotations

import torch
from torch import nn

from .initnet import context_features
from .unrolled import boundary_projection, device_constants_of


def latent_length(n: int) -> int:
    """L = 25 latent vectors for the 4- and 8-agent models, 100 for 16 agents and more."""
    return 25 if n <= 8 else 100


class StateNet(nn.Module):
    """Two convolution layers (ReLU, batch norm) over the 18 start/goal channels of each robot, max-pooled
    over the robots and broadcast along the latent positions."""

    def __init__(self, width: int = 64):
        super().__init__()
        self.net = nn.Sequential(nn.Conv1d(18, width, 1), nn.BatchNorm1d(width), nn.ReLU(),
                                 nn.Conv1d(width, width, 1), nn.BatchNorm1d(width), nn.ReLU())

    def forward(self, state: torch.Tensor, length: int) -> torch.Tensor:
        return self.net(state).amax(dim=2, keepdim=True).expand(-1, -1, length)


def _deconv_stack(c_in: int, act, dropout: float) -> nn.Sequential:
    layers = []
    for i in range(4):
        layers += [nn.ConvTranspose1d(c_in if i == 0 else 128, 128, kernel_size=3, padding=1), nn.BatchNorm1d(128),
                   act(), nn.Dropout(dropout)]
    return nn.Sequential(*layers)


class _Decoder(nn.Module):
    def __init__(self, n: int, m1: int, c_in: int, act, dropout: float, scale: float):
        super().__init__()
        self.n, self.m1, self.L, self.scale = n, m1, latent_length(n), scale
        self.body = _deconv_stack(c_in, act, dropout)
        self.head = nn.Conv1d(128, 3, 1)                         # 3 axes per latent position
        self.expand = nn.Linear(self.L, n * m1)                 # latent positions -> robot x coefficient

    def _coeffs(self, h: torch.Tensor) -> torch.Tensor:
        out = self.expand(self.head(self.body(h)))              # (B, 3, n m1)
        return self.scale * out.reshape(out.shape[0], -1)


class CVAEDecoder(_Decoder):
    """Gaussian latent (B, 3, L) + state features -> coefficient correction (B, 3 n m1)."""

    def __init__(self, n: int, m1: int = 11, state_width: int = 64, dropout: float = 0.1, scale: float = 0.5):
        super().__init__(n, m1, 3 + state_width, lambda: nn.LeakyReLU(0.01), dropout, scale)
        self.state = StateNet(state_width)

    def sample_latent(self, batch: int, generator: torch.Generator | None = None, device=None) -> torch.Tensor:
        return torch.randn((batch, 3, self.L), generator=generator, device=device)

    def forward(self, z: torch.Tensor, state: torch.Tensor) -> torch.Tensor:
        return self._coeffs(torch.cat([z, self.state(state, self.L)], dim=1))


class VQVAEDecoder(_Decoder):
    """Code indices (B, L) into a 512 x 3 codebook -> coefficient correction (B, 3 n m1)."""

    def __init__(self, n: int, m1: int = 11, codes: int = 512, dropout: float = 0.1, scale: float = 0.5):
        super().__init__(n, m1, 3, nn.ReLU, dropout, scale)
        self.codebook = nn.Embedding(codes, 3)

    def sample_latent(self, batch: int, generator: torch.Generator | None = None, device=None) -> torch.Tensor:
        return torch.randint(0, self.codebook.num_embeddings, (batch, self.L), generator=generator, device=device)

    def forward(self, idx: torch.Tensor, state: torch.Tensor | None = None) -> torch.Tensor:
        return self._coeffs(self.codebook(idx).transpose(1, 2))


@torch.no_grad()
def calibrate_batchnorm(sf, decoder: nn.Module, batches: int = 4, batch: int = 256, seed: int = 0) -> nn.Module:
    """Set the batch-norm running statistics of a random-init decoder from its own sampled latents
    (train-mode passes with a cumulative average), so the eval-mode decoder normalises its activations
    and the latent keeps its influence through the four layers."""
    dev = next(decoder.parameters()).device
    for m in decoder.modules():
        if isinstance(m, nn.modules.batchnorm._BatchNorm):
            m.reset_running_stats()
            m.momentum = None
    decoder.train()
    gen = torch.Generator(device=dev).manual_seed(seed)
    state = torch.as_tensor(context_features(sf.problem), dtype=torch.float32, device=dev)
    for _ in range(batches):
        decoder(decoder.sample_latent(batch, gen, dev), state.expand(batch, -1, -1))
    return decoder.eval()


def _tf32_split(x: torch.Tensor):
    """(hi, lo) float32 with hi = x rounded to tf32 (nearest, ties away: cvt.rna) and lo = tf32(x - hi)."""
    def rna(v):
        b = v.contiguous().view(torch.int32)
        return ((b + 0x1000) & ~0x1FFF).view(torch.float32)
    x = x.to(torch.float32)
    hi = rna(x)
    return hi, rna(x - hi)


class FusedDecoder:
    """The decoder's eval-mode forward pass as one sm_100a kernel (K4, ``sgsf_decoder_forward``): batch norm
    folded into the convolutions, weights packed once into the tensor-core operand layout (tf32 hi / lo per
    32 KB stage of (tap, 32 input channels)).  ``__call__(latent, state)`` returns what
    ``decoder(latent, state).to(float64)`` returns, computed on the tensor cores to FP32-level accuracy."""

    STAGE = 32768

    def __init__(self, decoder: nn.Module, device=None):
        from . import native
        self.decoder = decoder.eval()
        dev = torch.device(device) if device is not None else next(decoder.parameters()).device
        self.dev = dev
        convs = [m for m in decoder.body if isinstance(m, nn.ConvTranspose1d)]
        bns = [m for m in decoder.body if isinstance(m, nn.modules.batchnorm._BatchNorm)]
        acts = [m for m in decoder.body if isinstance(m, (nn.LeakyReLU, nn.ReLU))]
        assert len(convs) == 4 and len(bns) == 4 and all(c.kernel_size == (3,) and c.padding == (1,) for c in convs)
        self.leaky = isinstance(acts[0], nn.LeakyReLU)
        self.slope = float(acts[0].negative_slope) if self.leaky else 0.0
        self.c0 = convs[0].in_channels
        c0p = ((self.c0 + 31) // 32) * 32
        stages, biases = [], []
        with torch.no_grad():
            for li, (cv, bn) in enumerate(zip(convs, bns)):
                Wt = cv.weight.detach().double().cpu()                  # (c_in, c_out, 3)
                Wc = Wt.flip(2).permute(1, 0, 2).contiguous()          # conv form (c_out, c_in, tap)
                sc = bn.weight.double().cpu() / torch.sqrt(bn.running_var.double().cpu() + bn.eps)
                Wc = Wc * sc[:, None, None]
                b = (cv.bias.double().cpu() - bn.running_mean.double().cpu()) * sc + bn.bias.double().cpu()
                cin = Wc.shape[1]
                cinp = c0p if li == 0 else 128
                Wp = torch.zeros(128, cinp, 3, dtype=torch.float64)
                Wp[:, :cin] = Wc
                for tap in range(3):
                    for cg in range(cinp // 32):
                        blk = Wp[:, cg * 32:(cg + 1) * 32, tap].reshape(128, 8, 4).permute(1, 0, 2)  # [chunk][m][4]
                        hi, lo = _tf32_split(blk.float())
                        stages.append(torch.cat([hi.reshape(-1), lo.reshape(-1)]))
                biases.append(b.float())
        self.wpack = torch.cat(stages).to(dev).contiguous()
        assert self.wpack.numel() * 4 == native.load().sgsf_decoder_pack_bytes(self.c0)
        self.bias = torch.cat(biases).to(dev).contiguous()
        self.head_w = decoder.head.weight.detach().float().reshape(3, 128).to(dev).contiguous()
        self.head_b = decoder.head.bias.detach().float().to(dev).contiguous()
        self.exp_w = decoder.expand.weight.detach().float().t().to(dev).contiguous()   # (L, n m1): transposed
        self.exp_b = decoder.expand.bias.detach().float().to(dev).contiguous()
        self.L, self.nm1, self.scale = decoder.L, decoder.n * decoder.m1, float(decoder.scale)
        self._feat_key, self._feat = None, None
        self._descs: dict = {}

    def _desc(self, cz: int, feat, qp: dict | None):
        key = (cz, feat.data_ptr() if feat is not None else 0, id(qp))
        d = self._descs.get(key)
        if d is None:
            d = self._descs[key] = (self._make_desc(cz, feat, qp), qp)   # (qp kept alive: its id is the key)
        return d[0]

    def _make_desc(self, cz: int, feat, qp: dict | None):
        from . import native
        d = native.Decoder(self.L, self.c0, self.nm1, int(self.leaky), self.slope, self.scale,
                           self.wpack.data_ptr(), self.bias.data_ptr(), self.head_w.data_ptr(),
                           self.head_b.data_ptr(), self.exp_w.data_ptr(), self.exp_b.data_ptr(), cz,
                           feat.data_ptr() if feat is not None else None)
        if qp is not None:
            d.base, d.B6, d.PBt, d.rhs = (qp[k].data_ptr() for k in ("base", "B", "PBt", "rhs"))
            d.n, d.m1 = qp["n"], qp["m1"]
        return d

    @torch.no_grad()
    def state_features(self, state: torch.Tensor) -> torch.Tensor:
        """(c0 - 3,) float32: the CVAE's state-network features of one problem's start/goal context (the same
        for every sample), cached per context tensor."""
        key = (state.data_ptr(), tuple(state.shape))
        if self._feat_key != key:
            with torch.backends.cudnn.flags(enabled=True, allow_tf32=False):
                self._feat = self.decoder.state(state[:1].to(torch.float32), 1)[0, :, 0].contiguous()
            self._feat_key = key
        return self._feat

    @torch.no_grad()
    def first_layer_input(self, latent: torch.Tensor, state: torch.Tensor | None) -> torch.Tensor:
        """(B, c0, L) float32: the latent (CVAE: with the broadcast state features; VQ-VAE: codebook vectors)."""
        d = self.decoder
        if isinstance(d, CVAEDecoder):
            # one problem: the same features for all samples; full FP32 (cuDNN's default TF32 would put a 1e-3
            # relative error into every sample's input)
            with torch.backends.cudnn.flags(enabled=True, allow_tf32=False):
                feat = d.state(state[:1].to(torch.float32), d.L)
            return torch.cat([latent.to(torch.float32), feat.expand(latent.shape[0], -1, -1)], dim=1).contiguous()
        return d.codebook(latent).transpose(1, 2).contiguous()

    @torch.no_grad()
    def __call__(self, latent: torch.Tensor, state: torch.Tensor | None = None, qp: dict | None = None) -> torch.Tensor:
        """The correction ``decoder(latent, state)`` (B, 3 n m1) FP64; with ``qp`` (the QP layer's device
        constants: base, B, PBt, rhs, n, m1) the projected proposals boundary_projection(base + correction),
        with the QP layer fused into the kernel."""
        from . import native
        from .solver import _stream
        d = self.decoder
        if isinstance(d, CVAEDecoder):   # the latent per sample, the state features from a per-problem cache
            h0, feat, cz = latent.to(torch.float32).contiguous(), self.state_features(state), latent.shape[1]
        else:
            h0, feat, cz = d.codebook(latent).transpose(1, 2).contiguous(), None, self.c0
        B = int(h0.shape[0])
        out = torch.empty((B, 3 * self.nm1), dtype=torch.float64, device=h0.device)
        if B:
            desc = self._desc(cz, feat, qp)
            native.check(native.load().sgsf_decoder_forward(desc, B, h0.data_ptr(), out.data_ptr(), _stream()),
                         "sgsf_decoder_forward")
        return out


def make_decoder(kind: str, n: int, m1: int = 11, **kw) -> nn.Module:
    if kind == "cvae":
        return CVAEDecoder(n, m1, **kw)
    if kind == "vqvae":
        return VQVAEDecoder(n, m1, **kw)
    raise ValueError(f"decoder kind must be 'cvae' or 'vqvae', got {kind!r}")


def decode_proposals(sf, decoder: nn.Module, latent: torch.Tensor, fused: "FusedDecoder | None" = None) -> torch.Tensor:
    """xi_bar (B, dim) float64 on the decoder's device: the straight line plus the decoder's correction,
    through the boundary QP layer (projection.py:11-25).  With ``fused`` (a :class:`FusedDecoder` of the same
    decoder) the correction comes from the sm_100a decoder kernel K4 instead of the PyTorch module."""
    k = device_constants_of(sf, latent.device)
    state, base = k["context32"], k["base"]   # (one tensor per filter: the decoder's state-feature cache key)
    st = state.expand(latent.shape[0], -1, -1)
    if fused is not None:   # decoder + QP layer in one kernel
        return fused(latent, st, qp=k)
    return boundary_projection(sf, base + decoder(latent, st).to(torch.float64))


@torch.no_grad()
def generate_and_filter(sf, decoder: nn.Module, batch: int, seed: int = 0, init_net=None, config=None,
                        fused: "FusedDecoder | None" = None):
    """Sample ``batch`` proposals from the decoder and filter them, all on the current CUDA device (no host
    round trip): latent -> decoder (kernel K4 when ``fused`` is given) -> QP layer -> (init network) -> SF
    kernel.  Returns (xi_bar, DeviceBatch)."""
    dev = torch.device("cuda", torch.cuda.current_device())
    decoder.to(dev).eval()
    gen = torch.Generator(device=dev).manual_seed(seed)
    xb = decode_proposals(sf, decoder, decoder.sample_latent(batch, gen, dev), fused)
    xi0 = lam0 = None
    if init_net is not None:
        from .initnet import initial_states
        xi0, lam0 = initial_states(sf, xb, "initnet", init_net)
    return xb, sf.solve_batched(xb, xi0=xi0, lam0=lam0, config=config)


class PipelineGraph:
    """The whole generate-and-filter step (latent -> decoder -> QP layer -> [init net] -> SF kernel ->
    verdict) captured once as a CUDA graph and replayed.  Small batches (BASELINE config 1: 8 samples) are
    bound by the launch latency of the decoder's and the solve's few dozen kernels; a replay is one
    launch.  Inputs and outputs are static buffers: :meth:`replay` copies a new latent in and returns the
    same (xi_bar, DeviceBatch) tensors, overwritten."""

    def __init__(self, sf, decoder: nn.Module, batch: int, init_net=None, config=None, seed: int = 0,
                 warmup: int = 2, fused: bool = True):
        dev = torch.device("cuda", torch.cuda.current_device())
        self.sf, self.decoder, self.init_net, self.config = sf, decoder.to(dev).eval(), init_net, config
        self.fused = FusedDecoder(self.decoder) if fused else None
        if init_net is not None:
            init_net.to(dev).eval()
        gen = torch.Generator(device=dev).manual_seed(seed)
        self.latent = decoder.sample_latent(batch, gen, dev)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):   # lazy initialisation (handles, cuDNN plans) before the capture
            for _ in range(warmup):
                self._run()
        torch.cuda.current_stream().wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.xi_bar, self.out = self._run()

    @torch.no_grad()
    def _run(self):
        xb = decode_proposals(self.sf, self.decoder, self.latent, self.fused)
        xi0 = lam0 = None
        if self.init_net is not None:
            from .initnet import initial_states
            xi0, lam0 = initial_states(self.sf, xb, "initnet", self.init_net)
        return xb, self.sf.solve_batched(xb, xi0=xi0, lam0=lam0, config=self.config)

    def replay(self, latent: torch.Tensor | None = None):
        if latent is not None:
            self.latent.copy_(latent)
        self.graph.replay()
        return self.xi_bar, self.out
