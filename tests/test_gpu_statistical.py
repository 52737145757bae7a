"""Statistical pins of the GPU path at scale (SURVEY §8c "What pins each part"):

* token histogram (V = 1024): over many independent trials of one request
  (fixed target rows p_i and draft rows q_i, fresh draft tokens x_i ~ q_i and
  uniforms per trial), the FIRST emitted token -- x_0 if accepted, else the
  resampled token -- is distributed as p_0 (losslessness); chi^2
  at the 1 % level.  P(n >= 1) = beta_0 = sum_x min(p_0, q_0) within 4 sigma.
* Monte Carlo expected acceptance at the Qwen shape (V = 152064, gamma = 3):
  mean n over 2048 trials equals sum_{k=1..gamma} prod_{i<k} beta_i within 4 sigma
  (Leviathan's closed form; beta_i from the fp64 oracle rows).
The closed forms use the fp64 oracle's probabilities of the same bf16 inputs.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2512_22420_b200 import Verifier
from synth.inputs import make_batch, make_weight

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0") if torch.cuda.is_available() else None


def _trials(b0, gamma, B, nbatch, seed, W):
    """Replicate request 0 of b0 B times per batch with fresh x_i ~ q_i and uniforms."""
    V, d = W.shape
    g = torch.Generator(device=DEV)
    g.manual_seed(seed)
    H = b0.hidden[: gamma + 1]
    Q = b0.draft_probs[:gamma]
    v = Verifier(d, V, max_batch=B, gamma_max=gamma)
    hid = H.repeat(B, 1).contiguous()
    q = Q.repeat(B, 1).contiguous()
    gam = np.full(B, gamma, np.int32)
    acc = torch.empty(B, dtype=torch.int32, device=DEV)
    nxt = torch.empty(B, dtype=torch.int32, device=DEV)
    out_n, out_first = [], []
    for _ in range(nbatch):
        x = torch.multinomial(Q, B, replacement=True, generator=g).t().contiguous().view(-1).to(torch.int32)
        u = (torch.randint(0, 1 << 24, (B * (gamma + 1),), generator=g, device=DEV).double() * 2.0 ** -24).float()
        v.verify(hid, W, x, q, gam, u, acc, nxt)
        torch.cuda.synchronize()
        a = acc.cpu().numpy()
        x0 = x.view(B, gamma)[:, 0].cpu().numpy()
        out_n.append(a)
        out_first.append(np.where(a >= 1, x0, nxt.cpu().numpy()))
    return np.concatenate(out_n), np.concatenate(out_first)


def _oracle_rows(b0, gamma, W_bits):
    n = b0.to_numpy()
    r = oracle.verify(n["hidden_bits"][: gamma + 1], W_bits, n["draft_tokens"][:gamma],
                      n["draft_probs"][:gamma], np.array([gamma], np.int32), n["uniforms"][: gamma + 1])
    L = oracle.logits(n["hidden_bits"][: gamma + 1], W_bits)
    P = np.exp(L - r["lse"][:, None])
    return P, np.asarray(n["draft_probs"][:gamma], np.float64)


def test_first_token_law_chi2():
    from scipy.stats import chi2
    V, d, gamma = 1024, 64, 2
    W = make_weight(V, d, 3, DEV)
    b0 = make_batch(1, gamma, V=V, d=d, seed=4, device=DEV, W=W, sigma_n=1.0)
    P, Q = _oracle_rows(b0, gamma, b0.to_numpy()["W_bits"])
    n, first = _trials(b0, gamma, B=512, nbatch=100, seed=7, W=W)
    T = first.size
    obs = np.bincount(first, minlength=V).astype(np.float64)
    exp = P[0] * T
    big = exp >= 5.0
    o = np.concatenate([obs[big], [obs[~big].sum()]])
    e = np.concatenate([exp[big], [exp[~big].sum()]])
    keep = e > 0
    stat = float(((o[keep] - e[keep]) ** 2 / e[keep]).sum())
    dof = int(keep.sum()) - 1
    assert chi2.sf(stat, dof) > 0.01, (stat, dof)
    beta0 = np.minimum(P[0], Q[0]).sum()
    p_hat = float((n >= 1).mean())
    assert abs(p_hat - beta0) <= 4 * np.sqrt(beta0 * (1 - beta0) / T), (p_hat, beta0)


def test_expected_accept_length_qwen_shape():
    V, d, gamma = 152064, 3584, 3
    W = make_weight(V, d, 0, DEV)
    b0 = make_batch(1, gamma, V=V, d=d, seed=21, device=DEV, W=W, sigma_n=1.0)
    P, Q = _oracle_rows(b0, gamma, b0.to_numpy()["W_bits"])
    beta = [np.minimum(P[i], Q[i]).sum() for i in range(gamma)]
    closed = sum(np.prod(beta[:k]) for k in range(1, gamma + 1))
    n, _ = _trials(b0, gamma, B=256, nbatch=8, seed=11, W=W)
    se = n.std() / np.sqrt(n.size)
    assert abs(n.mean() - closed) <= 4 * se + 1e-9, (n.mean(), closed, se)
