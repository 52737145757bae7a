"""GPU parity of greedy verification nj_verify_greedy (
include/nj.h) against oracle.verify_greedy (fp64 argmax): accept_len and
next_token bit-exact except requests whose consulted rows have a top-2 logit
gap <= 1e-4 (counted, excused; fp32 logits error is ~1e-5 at most)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2512_22420_b200 import NJError, Verifier
from synth.inputs import make_batch, make_weight

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0") if torch.cuda.is_available() else None
QV, QD = 152064, 3584
_W = {}


def run(b, max_batch=None, tokens=None):
    v = Verifier(b.hidden.shape[1], b.W.shape[0], max_batch=max_batch or b.B, gamma_max=5)
    acc = torch.full((b.B,), -7, dtype=torch.int32, device=DEV)
    nxt = torch.full((b.B,), -7, dtype=torch.int32, device=DEV)
    v.verify_greedy(b.hidden, b.W, b.draft_tokens if tokens is None else tokens, b.gamma, acc, nxt)
    torch.cuda.synchronize()
    return acc.cpu().numpy(), nxt.cpu().numpy(), v


def check(b, acc, nxt, tokens=None):
    n = b.to_numpy()
    x = n["draft_tokens"] if tokens is None else tokens.cpu().numpy()
    r = oracle.verify_greedy(n["hidden_bits"], n["W_bits"], x, n["gamma"])
    ok = ~r["tie"]
    assert ((acc != r["accept_len"]) & ok).sum() == 0, (acc, r["accept_len"])
    assert ((nxt != r["next_token"]) & ok).sum() == 0, (nxt, r["next_token"])
    # excused requests (a consulted row's top-2 gap <= 1e-4): the GPU outcome must
    # follow from SOME choice of near-maximal tokens (within 1e-4 of the row max)
    if (~ok).any():
        L = oracle.logits(n["hidden_bits"], n["W_bits"])
        g = n["gamma"]
        ro = np.concatenate([[0], np.cumsum(g + 1)])
        near = lambda j, t: L[j, t] >= L[j].max() - 1e-4
        for bb in np.nonzero(~ok)[0]:
            a, t, r0, d0 = int(acc[bb]), int(nxt[bb]), ro[bb], ro[bb] - bb
            assert all(near(r0 + i, x[d0 + i]) for i in range(a)), bb
            assert near(r0 + a, t) and (a == g[bb] or t != x[d0 + a]), bb
    return r


@pytest.mark.parametrize("B,g,V,d", [(1, 3, 32, 16), (12, "mixed:5", 4099, 64), (40, 0, 2048, 128),
                                     (140, 3, 1000, 64)])
def test_greedy_small(B, g, V, d):
    """incl. gamma = 0 (plain greedy decoding) and N = 560 > 512 (two GEMM blocks)."""
    b = make_batch(B, g, V=V, d=d, seed=B + 1, device=DEV)
    acc, nxt, _ = run(b)
    check(b, acc, nxt)


def test_greedy_argmax_drafts_accepted_full_size():
    """Qwen shape: drafts that copy the target argmax are accepted in full and
    the bonus token is the last row's argmax; random drafts reject early."""
    if "W" not in _W:
        _W["W"] = make_weight(QV, QD, 0, DEV)
    b = make_batch(16, 3, V=QV, d=QD, seed=3, device=DEV, W=_W["W"])
    acc, nxt, _ = run(b)
    r = check(b, acc, nxt)
    a = torch.tensor(r["argmax"], dtype=torch.int32, device=DEV)
    rows = [ro + i for bb, ro in enumerate(range(0, 64, 4)) for i in range(3)]
    x = a[torch.tensor(rows, device=DEV)].contiguous()
    acc2, nxt2, _ = run(b, tokens=x)
    check(b, acc2, nxt2, tokens=x)
    assert (acc2 == 3).all()


def test_greedy_c3_mixed_full_size():
    if "W" not in _W:
        _W["W"] = make_weight(QV, QD, 0, DEV)
    b = make_batch(64, "mixed:5", V=QV, d=QD, seed=9, device=DEV, W=_W["W"])
    acc, nxt, _ = run(b)
    check(b, acc, nxt)


def test_greedy_errors():
    b = make_batch(4, 2, V=512, d=32, seed=1, device=DEV)
    v = Verifier(32, 512, max_batch=4, gamma_max=2)
    acc = torch.empty(4, dtype=torch.int32, device=DEV)
    with pytest.raises(NJError):   # gamma above gamma_max
        v.verify_greedy(b.hidden, b.W, b.draft_tokens, np.full(4, 3, np.int32), acc, acc)
    with pytest.raises(NJError):   # B above max_batch
        v.verify_greedy(b.hidden, b.W, b.draft_tokens, np.full(5, 0, np.int32), acc, acc)
