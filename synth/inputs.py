"""Seeded synthetic inputs for the verification path.

This module is shared by the oracle side (tests, cpu_baseline) and the CUDA
side (tests, bench).  It holds NONE of the verification method's arithmetic:
it only draws random tensors.  The synthetic *draft model* distribution q is
an input to the method (the draft forward is out of scope)
and is modelled here as a noisy, flattened copy of the target logits computed
with plain torch ops (torch.matmul / torch.softmax), which belong to neither
the oracle nor the CUDA path.

Workload shape (BJ configs; P:234 DeepSeek-R1-Distill-Qwen-7B + 0.5B draft):
  d = 3584, V = 152064, B in 1..256, gamma in 0..5.

Recipe:
  hidden  h_r = s_r * z,  z ~ N(0,1) iid,  s_r ~ LogUniform[0.6, 1.6], bf16
  W_lm    N(0, sigma_l^2 / d), sigma_l = 3, bf16            -> logit std 1.8-4.8
  q_i     softmax(tau_q * (l_hat_i + sigma_n * xi)), tau_q = 0.9, xi ~ N(0,1)
          l_hat = fp32 torch logits of the same bf16 inputs (setup only);
          optional q = 0 on ids >= q_vocab (draft vocabulary smaller than V)
  x_i     ~ q_i (torch.multinomial, own generator)       -> q_i(x_i) > 0
  u       randint(0, 2^24) * 2^-24 (fp32-exact, in [0,1))   (R4)
Every stream has its own generator seeded from (seed, stream id).
"""
from __future__ import annotations

import dataclasses

import numpy as np
import torch

QWEN7B_D = 3584
QWEN7B_V = 152064
DRAFT05B_V = 151936  # 0.5B draft vocabulary size (ext, model config)

_STREAMS = {"hidden": 1, "scale": 2, "W": 3, "noise": 4, "draft": 5, "uniform": 6, "gamma": 7}


def _gen(seed: int, stream: str, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed((int(seed) * 1_000_003 + _STREAMS[stream] * 7919) & 0x7FFF_FFFF_FFFF_FFFF)
    return g


@dataclasses.dataclass
class Batch:
    hidden: torch.Tensor        # [N, d] bf16
    W: torch.Tensor             # [V, d] bf16
    draft_tokens: torch.Tensor  # [G] int32
    draft_probs: torch.Tensor   # [G, V] fp32 (G >= 1 rows; a dummy row when G = 0)
    gamma: np.ndarray           # [B] int32 (host)
    uniforms: torch.Tensor      # [N] fp32

    @property
    def B(self):
        return int(self.gamma.shape[0])

    @property
    def N(self):
        return int(self.gamma.sum()) + self.B

    @property
    def G(self):
        return int(self.gamma.sum())

    def to_numpy(self):
        """Host copies for the oracle: bf16 as uint16 bits, exact."""
        return dict(
            hidden_bits=self.hidden.cpu().contiguous().view(torch.int16).numpy().view(np.uint16),
            W_bits=self.W.cpu().contiguous().view(torch.int16).numpy().view(np.uint16),
            draft_tokens=self.draft_tokens.cpu().numpy().astype(np.int32),
            draft_probs=self.draft_probs.cpu().numpy(),
            gamma=self.gamma.astype(np.int32),
            uniforms=self.uniforms.cpu().numpy(),
        )


def make_weight(V: int, d: int, seed: int = 0, device="cpu", sigma_l: float = 3.0) -> torch.Tensor:
    g = _gen(seed, "W", device)
    # chunked to bound fp32 scratch at full size (545M elements)
    step = max(1, (1 << 26) // max(d, 1))
    out = torch.empty((V, d), dtype=torch.bfloat16, device=device)
    for v0 in range(0, V, step):
        v1 = min(V, v0 + step)
        out[v0:v1] = (torch.randn((v1 - v0, d), generator=g, device=device)
                      * (sigma_l / d ** 0.5)).to(torch.bfloat16)
    return out


def make_gamma(B: int, gamma, seed: int = 0) -> np.ndarray:
    """gamma: int (uniform) or 'mixed:<gmax>' (gamma_b ~ U{0..gmax} iid)."""
    if isinstance(gamma, str) and gamma.startswith("mixed"):
        gmax = int(gamma.split(":")[1]) if ":" in gamma else 5
        rng = np.random.default_rng(seed * 7 + 11)
        return rng.integers(0, gmax + 1, size=B).astype(np.int32)
    if isinstance(gamma, (list, tuple, np.ndarray)):
        return np.asarray(gamma, np.int32)
    return np.full(B, int(gamma), np.int32)


def make_batch(B: int, gamma, V: int, d: int, seed: int = 0, device="cpu",
               W: torch.Tensor | None = None, sigma_n: float = 1.0, tau_q: float = 0.9,
               q_vocab: int | None = None, sigma_l: float = 3.0) -> Batch:
    gam = make_gamma(B, gamma, seed)
    N = int(gam.sum()) + B
    G = int(gam.sum())
    if W is None:
        W = make_weight(V, d, seed, device, sigma_l)
    gz = _gen(seed, "hidden", device)
    gs = _gen(seed, "scale", device)
    z = torch.randn((N, d), generator=gz, device=device)
    s = torch.exp(torch.empty((N, 1), device=device).uniform_(np.log(0.6), np.log(1.6), generator=gs))
    hidden = (z * s).to(torch.bfloat16)
    # draft rows: row_off(b) + i for i < gamma_b
    row_off = np.concatenate([[0], np.cumsum(gam + 1)[:-1]]).astype(np.int64)
    drows = np.concatenate([row_off[b] + np.arange(gam[b]) for b in range(B)]) if G else np.zeros(0, np.int64)
    if G:
        hd = hidden[torch.as_tensor(drows, device=device)].float()
        l_hat = torch.matmul(hd, W.float().t()) if V * d < (1 << 27) else _chunked_logits(hd, W)
        gn = _gen(seed, "noise", device)
        xi = torch.randn(l_hat.shape, generator=gn, device=device)
        q = torch.softmax(tau_q * (l_hat + sigma_n * xi), dim=1)
        if q_vocab is not None and q_vocab < V:
            q[:, q_vocab:] = 0.0
            q = q / q.sum(dim=1, keepdim=True)
        q = q.float().contiguous()
        gd = _gen(seed, "draft", device)
        x = torch.multinomial(q, 1, generator=gd)[:, 0].to(torch.int32)
    else:
        q = torch.zeros((1, V), dtype=torch.float32, device=device)
        x = torch.zeros(0, dtype=torch.int32, device=device)
    gu = _gen(seed, "uniform", device)
    u = (torch.randint(0, 1 << 24, (N,), generator=gu, device=device).to(torch.float64)
         * 2.0 ** -24).to(torch.float32)
    return Batch(hidden, W, x, q, gam, u)


def _chunked_logits(hd: torch.Tensor, W: torch.Tensor) -> torch.Tensor:
    out = torch.empty((hd.shape[0], W.shape[0]), dtype=torch.float32, device=hd.device)
    step = 1 << 15
    for v0 in range(0, W.shape[0], step):
        out[:, v0:v0 + step] = torch.matmul(hd, W[v0:v0 + step].float().t())
    return out


def make_sampler_case(B: int, V: int, seed: int = 0, device="cpu", frac_residual: float = 0.6):
    """Inputs for the stage-isolated sampler test: fp32 logits [B, V] (std ~3),
    residual flags, q rows (noisy softmax of the logits), final uniforms."""
    g = _gen(seed, "hidden", device)
    logits = torch.randn((B, V), generator=g, device=device) * 3.0
    gn = _gen(seed, "noise", device)
    q = torch.softmax(0.9 * (logits + torch.randn((B, V), generator=gn, device=device)), dim=1).float()
    gr = _gen(seed, "gamma", device)
    residual = (torch.rand((B,), generator=gr, device=device) < frac_residual).to(torch.int32)
    gu = _gen(seed, "uniform", device)
    u = (torch.randint(0, 1 << 24, (B,), generator=gu, device=device).to(torch.float64)
         * 2.0 ** -24).to(torch.float32)
    return logits.contiguous(), residual, q.contiguous(), u


def qps_ramp(steps: int = 4000, qps_lo: float = 5.0, qps_hi: float = 300.0, bmax: int = 256,
             seed: int = 0) -> np.ndarray:
    """Config-4 batch-size trace: QPS rises linearly lo->hi over steps/2 then
    falls back (shape of fig:trace1; S:383-391 piecewise rate);
    B_t = clamp(round(QPS_t * bmax/qps_hi * (1 + 0.1 xi_t)), 1, bmax)."""
    half = steps // 2
    up = np.linspace(qps_lo, qps_hi, half)
    qps = np.concatenate([up, up[::-1]])[:steps]
    rng = np.random.default_rng(seed + 4242)
    B = np.rint(qps * bmax / qps_hi * (1.0 + 0.1 * rng.standard_normal(qps.shape[0])))
    return np.clip(B, 1, bmax).astype(np.int32)


def dyadic_rows(q: np.ndarray, bits: int = 20, min_count: int = 1) -> np.ndarray:
    """Round probability rows to k * 2^-bits with sum_x k = 2^bits exactly, so
    every row sums to exactly 1 in fp32 AND fp64 (R8: brute force
    uses exactly normalised q).  Entries keep at least min_count counts."""
    q = np.asarray(q, np.float64)
    total = 1 << bits
    out = np.empty_like(q, dtype=np.float32)
    for r in range(q.shape[0]):
        k = np.maximum(np.floor(q[r] / q[r].sum() * total), min_count).astype(np.int64)
        k[int(np.argmax(k))] += total - int(k.sum())
        assert k.min() >= 0 and int(k.sum()) == total
        out[r] = (k.astype(np.float64) / total).astype(np.float32)
    return out
