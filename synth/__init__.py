"""Seeded synthetic inputs shared by tests, bench and smoke.

This module holds NO arithmetic of the PASA method (no pooling, scoring,
routing, statistics, softmax or budget): it only draws the Q/K/V tensors and
latent trajectories that both the CUDA path and the oracle consume.  Recipes
are stated in DESIGN.md §5.

* ``iid_qkv``      -- Q, K, V ~ N(0, 1) (throughput configs; work is fixed by k).
* ``video_qkv``    -- tokens on the latent (F, H', W') patch grid with smooth
                      low-frequency structure, Q = K + 0.5 N, V = N + 0.5 K
                      (parity/fidelity: routing is non-trivial, attention local).
* ``three_phase``  -- flow-matching latent trajectory whose velocity noise has the
                      three-phase shape of PAPER.md:272-273 (high for the first
                      10 steps, low mid-trajectory, resurgent over the last 5).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

# BASELINE.json configs: (name, B, F, H', W', heads, D, latent shape)
CONFIGS = {
    "tiny": dict(B=1, S=1024, H=1, D=64, Bq=64, Bk=64, G=32, rho=0.5, grid=(1, 32, 32),
                 latent=(16, 4, 8, 8)),
    "tiny_g4": dict(B=1, S=1024, H=1, D=64, Bq=64, Bk=64, G=4, rho=0.5, grid=(1, 32, 32),
                    latent=(16, 4, 8, 8)),
    "wan13b_480p": dict(B=1, S=32760, H=12, D=128, Bq=128, Bk=64, G=32, rho=0.15,
                        grid=(21, 30, 52), latent=(16, 21, 60, 104)),
    "cogvideox5b": dict(B=1, S=17550, H=48, D=64, Bq=128, Bk=64, G=32, rho=0.15,
                        grid=(13, 30, 45), latent=(16, 13, 60, 90)),
    "wan14b_720p": dict(B=1, S=75600, H=40, D=128, Bq=128, Bk=64, G=32, rho=0.15,
                        grid=(21, 45, 80), latent=(16, 21, 90, 160)),
    "hunyuan_720p": dict(B=1, S=118800, H=24, D=128, Bq=128, Bk=64, G=32, rho=0.15,
                         grid=(33, 45, 80), latent=(16, 33, 90, 160)),
}


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def iid_qkv(B, S, H, D, *, seed=1000, dtype=torch.bfloat16, device="cpu"):
    g = _gen(seed, device)
    out = []
    for _ in range(3):
        out.append(torch.randn((B, S, H, D), generator=g, device=device, dtype=torch.float32)
                   .to(dtype))
    return tuple(out)


def video_qkv(B, grid, H, D, *, seed=7, dtype=torch.bfloat16, device="cpu", n_modes=8,
              noise=0.3):
    """Smooth video-like K on the (F, H', W') grid; S = F*H'*W', token index
    (f*H' + y)*W' + x.  Per (b, h, channel): sum of n_modes cosines with
    |omega| <= pi/4 per axis, unit RMS, plus ``noise``*N(0,1)."""
    F, Hp, Wp = grid
    S = F * Hp * Wp
    g = _gen(seed, device)
    f = torch.arange(F, device=device, dtype=torch.float32)
    y = torch.arange(Hp, device=device, dtype=torch.float32)
    x = torch.arange(Wp, device=device, dtype=torch.float32)
    ff, yy, xx = torch.meshgrid(f, y, x, indexing="ij")
    pos = torch.stack([ff.reshape(-1), yy.reshape(-1), xx.reshape(-1)], -1)  # [S, 3]
    K = torch.empty((B, S, H, D), device=device, dtype=torch.float32)
    for b in range(B):
        for h in range(H):
            om = (torch.rand((D, n_modes, 3), generator=g, device=device) * 2 - 1) * (math.pi / 4)
            ph = torch.rand((D, n_modes), generator=g, device=device) * (2 * math.pi)
            amp = torch.randn((D, n_modes), generator=g, device=device)
            arg = torch.einsum("sk,dmk->sdm", pos, om) + ph  # [S, D, M]
            kh = (amp * torch.cos(arg)).sum(-1)  # [S, D]
            kh = kh / kh.pow(2).mean(0, keepdim=True).sqrt().clamp_min(1e-6)
            K[b, :, h, :] = kh
    K = K + noise * torch.randn(K.shape, generator=g, device=device)
    Q = K + 0.5 * torch.randn(K.shape, generator=g, device=device)
    V = torch.randn(K.shape, generator=g, device=device) + 0.5 * K
    return Q.to(dtype), K.to(dtype), V.to(dtype)


def correlated_qkv(B, S, H, D, *, strength=1.0, Bk=64, seed=7, dtype=torch.bfloat16,
                   device="cpu", spread=0.5):
    """SPEC.md:546 correlated-block generator: keys of KV block j are a shared
    anchor a_j plus ``spread``*N(0,1) deviations; V rows are ``strength`` times a
    fixed random linear map of the key deviation plus (1-strength)*N(0,1), so the
    within-block K-V covariance H_j (Eq. 5) is large; Q rows lean towards their
    own block's anchor (local attention).  strength in [0, 1]."""
    g = _gen(seed, device)
    NK = (S + Bk - 1) // Bk
    blk = torch.arange(S, device=device) // Bk
    anchor = torch.randn((B, NK, H, D), generator=g, device=device)
    dev = spread * torch.randn((B, S, H, D), generator=g, device=device)
    K = anchor[:, blk] + dev
    M = torch.randn((H, D, D), generator=g, device=device) / math.sqrt(D)
    V = strength * torch.einsum("bshd,hde->bshe", dev / spread, M) \
        + (1.0 - strength) * torch.randn((B, S, H, D), generator=g, device=device)
    Q = 0.7 * anchor[:, blk] + 0.7 * torch.randn((B, S, H, D), generator=g, device=device)
    return Q.to(dtype), K.to(dtype), V.to(dtype)


@dataclass
class ThreePhase:
    """v_t = vbar + a_t xi_t, x_{t+1} = x_t + h v_t, h = 1/T, a_t = 3.0 (t < 10),
    0.5 (10 <= t < T-5), 2.0 (t >= T-5); x_0, vbar, xi_t ~ N(0,1) seeded."""
    shape: tuple
    T: int = 50
    seed: int = 7
    device: str = "cpu"
    a_early: float = 3.0
    a_mid: float = 0.5
    a_late: float = 2.0

    def amp(self, t: int) -> float:
        if t < 10:
            return self.a_early
        if t >= self.T - 5:
            return self.a_late
        return self.a_mid

    def latents(self, t: int):
        """Returns (x_t, x_{t-1}, x_{t-2}) as fp32 tensors (t >= 2)."""
        assert 2 <= t <= self.T
        g = _gen(self.seed, self.device)
        x = torch.randn(self.shape, generator=g, device=self.device)
        vbar = torch.randn(self.shape, generator=g, device=self.device)
        h = 1.0 / self.T
        hist = [x]
        for s in range(t):
            xi = torch.randn(self.shape, generator=g, device=self.device)
            x = x + h * (vbar + self.amp(s) * xi)
            hist.append(x)
            hist = hist[-3:]
        return hist[-1], hist[-2], hist[-3]

    def trajectory(self):
        """Yields x_0, x_1, ..., x_T in order (the same draws as latents(t))."""
        g = _gen(self.seed, self.device)
        x = torch.randn(self.shape, generator=g, device=self.device)
        vbar = torch.randn(self.shape, generator=g, device=self.device)
        h = 1.0 / self.T
        yield x
        for s in range(self.T):
            xi = torch.randn(self.shape, generator=g, device=self.device)
            x = x + h * (vbar + self.amp(s) * xi)
            yield x

    def expected_l1_offline(self, t: int) -> float:
        """E|v_t - v_{t-1}| (the paper's offline signal between adjacent steps)."""
        a1, a2 = self.amp(t), self.amp(t - 1)
        return math.sqrt(2.0 / math.pi) * math.sqrt(a1 * a1 + a2 * a2)

    def expected_l1(self, t: int) -> float:
        """E|v_{t-1} - v_{t-2}| for the online reading R-16 (closed form)."""
        a1, a2 = self.amp(t - 1), self.amp(t - 2)
        return math.sqrt(2.0 / math.pi) * math.sqrt(a1 * a1 + a2 * a2)

    def expected_l1_mean(self, dense_frac: float = 0.2) -> float:
        D = int(math.floor(dense_frac * self.T + 0.5))
        vals = [self.expected_l1(t) for t in range(max(D, 2), self.T)]
        return sum(vals) / len(vals)
