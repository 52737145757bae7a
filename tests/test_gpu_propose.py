"""GPU parity of the draft-side proposal step nj_propose (SURVEY §8(f) NEXT
row 1; include/nj.h): tokens x_b ~ q_b = softmax(W h_b) by inverse CDF with the
supplied uniforms, and the q rows it writes, against oracle.propose (fp64).
Bar as for verification (R12 / R16): tokens bit-exact outside the
1e-6 draw-tie band; |ln q_gpu - ln q_oracle| <= 2e-5 on q > 1e-30 (the staged
path's bound, same GEMM); q_b(x_b) > 0; rows sum to 1 within 1e-4."""
import numpy as np
import pytest
import torch

import oracle
import parity
from paper_2512_22420_b200 import NJError, Verifier
from synth.inputs import make_batch, make_weight

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0") if torch.cuda.is_available() else None
DV, DD = 151936, 896   # 0.5B-style draft head
_W = {}


def run(b, ldq=None):
    B, V = b.B, b.W.shape[0]
    v = Verifier(b.hidden.shape[1], V, max_batch=B, gamma_max=1)
    tok = torch.full((B,), -7, dtype=torch.int32, device=DEV)
    q = torch.full((B, ldq or V), float("nan"), device=DEV)
    v.propose(b.hidden, b.W, b.uniforms, tok, q[:, :V] if ldq else q)
    torch.cuda.synchronize()
    return tok.cpu().numpy(), q[:, :V].cpu().numpy().astype(np.float64), v


def check(b, tok, q, lnq_tol=2e-5):
    """Tokens via tests/parity.py (nj_propose is the gamma = 0 draw of q:
    bit-exact outside the 1e-6 band, excused draws must be a neighbour across
    the tied CDF boundary, excused count vs sum p_tie); q rows vs fp64."""
    import os
    n = b.to_numpy()
    r = oracle.propose(n["hidden_bits"], n["W_bits"], n["uniforms"])
    V = b.W.shape[0]
    nv = {"hidden_bits": n["hidden_bits"], "W_bits": n["W_bits"], "draft_tokens": np.zeros(0, np.int32),
          "draft_probs": np.zeros((1, V), np.float32), "gamma": np.zeros(b.B, np.int32), "uniforms": n["uniforms"]}
    parity.check(os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0], nv, np.zeros(b.B, np.int32), tok)
    assert (q[np.arange(b.B), tok] > 0).all()
    m = r["q"] > 1e-30
    err = np.abs(np.log(np.maximum(q[m], 1e-45)) - np.log(r["q"][m]))
    assert err.max(initial=0) <= lnq_tol, err.max()
    assert np.abs(q.sum(axis=1) - 1.0).max() <= 1e-4
    return int(r["tie"].sum())


@pytest.mark.parametrize("B,V,d", [(1, 32, 16), (3, 32, 16), (10, 4099, 64), (300, 2048, 128)])
def test_propose_small(B, V, d):
    for seed in range(2):
        b = make_batch(B, 0, V=V, d=d, seed=seed + 60, device=DEV)
        tok, q, _ = run(b)
        check(b, tok, q)


@pytest.mark.parametrize("B", [8, 64])
def test_propose_draft_shape(B):
    """0.5B-style draft head (d = 896, V = 151936), every position vs the oracle."""
    if "W" not in _W:
        _W["W"] = make_weight(DV, DD, 9, DEV)
    b = make_batch(B, 0, V=DV, d=DD, seed=B, device=DEV, W=_W["W"])
    tok, q, _ = run(b)
    check(b, tok, q)


def test_propose_strided_q_and_errors():
    b = make_batch(6, 0, V=1000, d=64, seed=3, device=DEV)
    tok, q, v = run(b, ldq=1003)
    check(b, tok, q)
    t = torch.empty(6, dtype=torch.int32, device=DEV)
    with pytest.raises(NJError):   # ldq < V
        v.propose(b.hidden, b.W, b.uniforms, t, torch.empty(6, 999, device=DEV))
    with pytest.raises(NJError):   # B > max_batch
        v.propose(torch.cat([b.hidden, b.hidden]), b.W, torch.cat([b.uniforms, b.uniforms]),
                  torch.empty(12, dtype=torch.int32, device=DEV), torch.empty(12, 1000, device=DEV))


def test_propose_then_verify_roundtrip():
    """The proposed (x, q) feed nj_verify directly: with the target = the draft
    (same W, same hidden), p = q, so every drafted token is accepted
    (u q < p fails only at u -> 1; PAPER.md:23 Leviathan acceptance)."""
    V, d, B, g = 2048, 64, 16, 3
    W = make_weight(V, d, 4, DEV)
    b = make_batch(B, g, V=V, d=d, seed=8, device=DEV, W=W)
    rows = torch.tensor([r for bb in range(B) for r in range(bb * (g + 1), bb * (g + 1) + g)], device=DEV)
    hd = b.hidden[rows].contiguous()
    vp = Verifier(d, V, max_batch=B * g, gamma_max=1)
    x = torch.empty(B * g, dtype=torch.int32, device=DEV)
    q = torch.empty(B * g, V, device=DEV)
    vp.propose(hd, W, b.uniforms[rows].contiguous(), x, q)
    vv = Verifier(d, V, max_batch=B, gamma_max=5)
    acc = torch.empty(B, dtype=torch.int32, device=DEV); nxt = torch.empty(B, dtype=torch.int32, device=DEV)
    u = torch.full_like(b.uniforms, 0.5)
    vv.verify(b.hidden, W, x, q, b.gamma, u, acc, nxt)
    torch.cuda.synchronize()
    assert (acc.cpu().numpy() == g).all()
