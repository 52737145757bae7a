"""GPU parity of the vocab-sharded mode (BJ config 5).

The per-rank kernels run inside an nj_group (G shards on one device, exchanges
as device copies) -- the only multi-shard setting one GPU allows -- and, for
the NCCL glue, as a single-rank NCCL communicator.  Bar as in
test_gpu_parity.py: accept_len / next_token equal the fp64 oracle (the
UNSHARDED definition) except in the 1e-6 tie band; ln p within 2e-3.
"""
import numpy as np
import pytest
import torch

import oracle
import parity
from paper_2512_22420_b200 import (NJ_FLAG_FALLBACK, NJ_OPT_CERTIFY, NJ_OPT_FORCE_FALLBACK, NJ_OPT_PATH, NJ_PATH_AUTO,
                                   NJ_PATH_TWOPASS, NcclComm, NJError, ShardGroup, Verifier, nccl_unique_id,
                                   shard_range)
from synth.inputs import make_batch, make_weight

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0") if torch.cuda.is_available() else None
QV, QD = 152064, 3584


def run_group(b, G, certify=True, force_fb=False, gamma_max=5, path=NJ_PATH_AUTO):
    """AUTO = the staged sharded step (k_lmhead over all rows of each shard) for
    N <= 2048; NJ_PATH_TWOPASS = the K-A / K-C form."""
    grp = ShardGroup(b.hidden.shape[1], b.W.shape[0], max_batch=b.B, gamma_max=gamma_max, nshards=G)
    grp.set_option(NJ_OPT_PATH, path)
    grp.set_option(NJ_OPT_CERTIFY, int(certify))
    grp.set_option(NJ_OPT_FORCE_FALLBACK, int(force_fb))
    acc = torch.full((b.B,), -7, dtype=torch.int32, device=DEV)
    nxt = torch.full((b.B,), -7, dtype=torch.int32, device=DEV)
    dd = {"lse": torch.full((b.N,), float("nan"), device=DEV), "p_draft": torch.zeros(max(b.G, 1), device=DEV),
          "mass": torch.zeros(b.B, dtype=torch.float64, device=DEV),
          "flags": torch.zeros(b.B, dtype=torch.int32, device=DEV)}
    grp.verify(b.hidden, grp.shards(b.W), b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt, debug=dd)
    torch.cuda.synchronize()
    return acc.cpu().numpy(), nxt.cpu().numpy(), {k: t.cpu().numpy() for k, t in dd.items()}


def check(b, acc, nxt, dd, lnp_tol=2e-3, name=None, L=None, n=None):
    """Decisions against the UNSHARDED oracle via tests/parity.py (band-aware,
    excused requests validity-checked and counted); p_draft and W_b against the
    oracle's fp64 values.  Returns the number of oracle ties."""
    import os
    name = name or os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]
    n = n or b.to_numpy()
    if L is None:
        L = (oracle.logits_blas(n["hidden_bits"], n["W_bits"]) if b.N >= 64 and b.W.shape[0] > 100000
             else oracle.logits(n["hidden_bits"], n["W_bits"]))
    r = parity.check(name, n, acc, nxt, gpu_flags=dd.get("flags"), L=L, certified=True)
    assert ((nxt >= 0) & (nxt < b.W.shape[0])).all()
    if b.G and "p_draft" in dd:
        m = r["p_draft"] > 1e-20
        lnp = np.abs(np.log(np.maximum(dd["p_draft"][:b.G][m], 1e-38)) - np.log(r["p_draft"][m]))
        assert lnp.max(initial=0) <= lnp_tol
    if "mass" in dd:
        same = (acc == r["accept_len"]) & ~((r["flags"] & oracle.F_ZERO_MASS) != 0)
        if same.any():
            assert np.abs(dd["mass"][same] - r["mass"][same]).max() <= 2e-5
    return int(r["tie"].sum())


def test_shard_ranges_partition():
    for V, G in [(QV, 2), (QV, 4), (QV, 8), (1000, 3), (2048, 8), (129, 2)]:
        rs = [shard_range(V, G, r) for r in range(G)]
        assert rs[0][0] == 0 and rs[-1][1] == V
        assert all(rs[i][1] == rs[i + 1][0] for i in range(G - 1))
        assert all(vb % 128 == 0 and ve > vb for vb, ve in rs)


@pytest.mark.parametrize("path", [NJ_PATH_AUTO, NJ_PATH_TWOPASS])
@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_group_small(G, path):
    for seed in range(3):
        b = make_batch(12, "mixed:5", V=2048, d=128, seed=40 + seed, device=DEV, q_vocab=2040)
        acc, nxt, dd = run_group(b, G, path=path)
        check(b, acc, nxt, dd, lnp_tol=2e-5)


@pytest.mark.parametrize("V,d,G", [(1000, 64, 3), (777, 40, 2), (4096, 256, 8)])
def test_group_ragged_vocab(V, d, G):
    b = make_batch(9, "mixed:4", V=V, d=d, seed=V, device=DEV, q_vocab=max(1, V - 5))
    acc, nxt, dd = run_group(b, G)
    check(b, acc, nxt, dd)


def test_group_equals_unsharded_gpu():
    """Sharded and unsharded GPU runs on identical inputs agree bit-exactly on
    the decisions (SURVEY §8e parity); here with all gamma = 0 (plain AR) too."""
    for B, g in [(40, "mixed:5"), (30, 0)]:
        b = make_batch(B, g, V=8192, d=512, seed=B, device=DEV)
        v = Verifier(512, 8192, max_batch=B, gamma_max=5)
        acc0 = torch.empty(B, dtype=torch.int32, device=DEV)
        nxt0 = torch.empty(B, dtype=torch.int32, device=DEV)
        v.verify(b.hidden, b.W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc0, nxt0)
        acc, nxt, dd = run_group(b, 4)
        ties = check(b, acc, nxt, dd)
        if ties == 0:
            assert (acc == acc0.cpu().numpy()).all() and (nxt == nxt0.cpu().numpy()).all()


@pytest.mark.parametrize("path", [NJ_PATH_AUTO, NJ_PATH_TWOPASS])
def test_group_forced_fp64_fallback(path):
    """Every request through the sharded fp64 fallback (three more exchanges)."""
    for G in (2, 4):
        b = make_batch(10, "mixed:3", V=2048, d=64, seed=21 + G, device=DEV)
        acc, nxt, dd = run_group(b, G, force_fb=True, path=path)
        check(b, acc, nxt, dd)
        assert (dd["flags"] & NJ_FLAG_FALLBACK).all()


def test_group_c5_full_size():
    """C5 shape per rank (G=8, gamma=2) at the Qwen vocabulary; B=32."""
    W = make_weight(QV, QD, 0, DEV)
    b = make_batch(32, 2, V=QV, d=QD, seed=55, device=DEV, W=W)
    acc, nxt, dd = run_group(b, 8)
    check(b, acc, nxt, dd, lnp_tol=4e-5)   # sharded K-A restarts every 14 k-blocks (certified)


@pytest.mark.parametrize("G,path", [(8, NJ_PATH_AUTO), (2, NJ_PATH_AUTO), (8, NJ_PATH_TWOPASS)])
def test_group_c5_bench_batch(G, path):
    """BASELINE configs[4] exactly: B = 256, gamma = 2 (N = 768) split over G
    vocab shards (the staged sharded step, and the two-pass form at G = 8),
    every request against the (unsharded) oracle."""
    W = make_weight(QV, QD, 0, DEV)
    b = make_batch(256, 2, V=QV, d=QD, seed=0, device=DEV, W=W)
    acc, nxt, dd = run_group(b, G, path=path)
    check(b, acc, nxt, dd, lnp_tol=4e-5, name=f"c5 bench batch G={G} path={path}")


def test_nccl_single_rank():
    """The NCCL glue of the sharded path with a one-rank communicator."""
    comm = NcclComm(1, nccl_unique_id(), 0, 0)
    try:
        b = make_batch(16, "mixed:5", V=4096, d=128, seed=3, device=DEV)
        v = Verifier(128, 4096, max_batch=16, gamma_max=5, nccl_comm=comm.handle)
        acc = torch.empty(16, dtype=torch.int32, device=DEV)
        nxt = torch.empty(16, dtype=torch.int32, device=DEV)
        p = torch.zeros(b.G, device=DEV)
        v.verify(b.hidden, b.W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt, debug={"p_draft": p})
        torch.cuda.synchronize()
        check(b, acc.cpu().numpy(), nxt.cpu().numpy(), {"p_draft": p.cpu().numpy()})
        with pytest.raises(NJError):   # a shard that is not nj_shard_range's
            Verifier(128, 4096, max_batch=16, gamma_max=5, nccl_comm=comm.handle, v_begin=128)
        v.close()
    finally:
        comm.close()


def test_group_large_batch_multi_launch():
    """G = 2000 draft rows: the sharded K-A spans two launches on every shard."""
    b = make_batch(400, 5, V=2048, d=64, seed=77, device=DEV)
    acc, nxt, dd = run_group(b, 4)
    check(b, acc, nxt, dd)
