"""GPU parity of the temperature variant (include/nj.h
nj_set_temperature): target p = softmax(l / T) on every path (fused, staged,
two-pass, vocab-sharded group, proposal) against the oracle at the same
temperature (oracle.verify(..., temperature=T), pinned to the T = 1 path by
test_temperature_power_of_two_equals_scaled_weights).  Bar as
test_gpu_parity.py (tests/parity.py: exact outside the 1e-6 band, excused
requests on a tie branch, counts bounded)."""
import os

import numpy as np
import pytest
import torch

import oracle
import parity
from paper_2512_22420_b200 import (NJ_OPT_CERTIFY, NJ_OPT_PATH, NJ_PATH_FUSED, NJ_PATH_STAGED, NJ_PATH_TWOPASS,
                                   NJError, ShardGroup, Verifier)
from synth.inputs import make_batch, make_weight

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0") if torch.cuda.is_available() else None
QV, QD = 152064, 3584


def _name():
    return os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]


def run(b, T, path, certify=True):
    v = Verifier(b.hidden.shape[1], b.W.shape[0], max_batch=b.B, gamma_max=5)
    v.set_option(NJ_OPT_PATH, path)
    v.set_option(NJ_OPT_CERTIFY, int(certify))
    v.set_temperature(T)
    acc = torch.full((b.B,), -7, dtype=torch.int32, device=DEV)
    nxt = torch.full((b.B,), -7, dtype=torch.int32, device=DEV)
    pd = torch.zeros(max(b.G, 1), device=DEV)
    fl = torch.zeros(b.B, dtype=torch.int32, device=DEV)
    v.verify(b.hidden, b.W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt,
             debug={"p_draft": pd, "flags": fl})
    torch.cuda.synchronize()
    return acc.cpu().numpy(), nxt.cpu().numpy(), pd.cpu().numpy(), fl.cpu().numpy()


def check(b, T, acc, nxt, pd, fl, lnp_tol=2e-3):
    n = b.to_numpy()
    if b.W.shape[0] == QV and b.N >= 64:
        L = oracle.logits_blas(n["hidden_bits"], n["W_bits"]) / T
    else:
        L = oracle.logits(n["hidden_bits"], n["W_bits"]) / T
    r = parity.check(f"{_name()} T={T}", n, acc, nxt, gpu_flags=fl, L=L)
    if b.G:
        m = r["p_draft"] > 1e-20
        lnp = np.abs(np.log(np.maximum(pd[:b.G][m], 1e-38)) - np.log(r["p_draft"][m]))
        assert lnp.max(initial=0) <= lnp_tol, lnp.max(initial=0)


@pytest.mark.parametrize("T", [0.5, 0.7, 2.0])
@pytest.mark.parametrize("path,B,g", [(NJ_PATH_FUSED, 8, "mixed:5"), (NJ_PATH_STAGED, 40, "mixed:5"),
                                      (NJ_PATH_TWOPASS, 40, "mixed:5")])
def test_temperature_paths(T, path, B, g):
    for seed in range(2):
        b = make_batch(B, g, V=4096, d=256, seed=seed + 3, device=DEV)
        acc, nxt, pd, fl = run(b, T, path)
        check(b, T, acc, nxt, pd, fl)


@pytest.mark.parametrize("T,B,g", [(0.7, 8, 3), (0.7, 64, 3), (1.5, 256, 2)])
def test_temperature_full_size(T, B, g):
    """Qwen shape on the fused (C2), staged and two-pass paths, certificate on
    and off."""
    W = make_weight(QV, QD, 0, DEV)
    b = make_batch(B, g, V=QV, d=QD, seed=B + 7, device=DEV, W=W)
    for certify in (True, False):
        acc, nxt, pd, fl = run(b, T, 0, certify=certify)
        check(b, T, acc, nxt, pd, fl, lnp_tol=5e-5)


def test_temperature_sharded_group():
    b = make_batch(12, "mixed:5", V=2048, d=128, seed=44, device=DEV, q_vocab=2040)
    grp = ShardGroup(128, 2048, max_batch=12, gamma_max=5, nshards=4)
    grp.set_temperature(0.6)
    acc = torch.empty(12, dtype=torch.int32, device=DEV)
    nxt = torch.empty(12, dtype=torch.int32, device=DEV)
    fl = torch.zeros(12, dtype=torch.int32, device=DEV)
    grp.verify(b.hidden, grp.shards(b.W), b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt,
               debug={"flags": fl})
    torch.cuda.synchronize()
    check(b, 0.6, acc.cpu().numpy(), nxt.cpu().numpy(), np.ones(max(b.G, 1)), fl.cpu().numpy(), lnp_tol=np.inf)


def test_temperature_propose_and_errors():
    b = make_batch(20, 0, V=3000, d=64, seed=9, device=DEV)
    v = Verifier(64, 3000, max_batch=20, gamma_max=1)
    v.set_temperature(0.8)
    tok = torch.empty(20, dtype=torch.int32, device=DEV)
    q = torch.empty(20, 3000, device=DEV)
    v.propose(b.hidden, b.W, b.uniforms, tok, q)
    torch.cuda.synchronize()
    n = b.to_numpy()
    r = oracle.propose(n["hidden_bits"], n["W_bits"], n["uniforms"], temperature=0.8)
    ok = ~r["tie"]
    assert (tok.cpu().numpy()[ok] == r["tokens"][ok]).all()
    qq = q.cpu().numpy().astype(np.float64)
    m = r["q"] > 1e-30
    assert np.abs(np.log(np.maximum(qq[m], 1e-45)) - np.log(r["q"][m])).max() <= 2e-5
    for bad in (0.0, -1.0, float("nan"), 1e7):
        with pytest.raises(NJError):
            v.set_temperature(bad)
