"""Reference of the vocab-sharded exchange protocol (NumPy fp64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  It writes out, rank by
rank, the decomposition that libnj's sharded mode uses (include/nj.h
"vocab-sharded mode") so that a real multi-rank
run over torch.distributed (gloo on CPU) can check the protocol's arithmetic
against the unsharded definition (oracle.verify):

  rank r owns vocab ids [v_r, v_{r+1}) (contiguous, rank order = ascending id);
  X1  per draft row:  (lse_r = log sum_{x in shard} e^{l(x)},  l(x_i) if owned)
      lse = log sum_r e^{lse_r}  (exact identity: the softmax normaliser is a
      sum over the partition of the vocabulary);
  X2  per request:    (lse used, W_r = sum_{x in shard} w(x), lse_r(n)) with w the
      residual max(0, p_n - q_n) (global lse) or the bonus p_gamma with the
      rank-local lse (so A_r = W_r e^{lse_r - M} are proportional to the shard
      masses); lse_r(n) is the shard's log-sum-exp of row n;
  R6  if sum_r W_r == 0 (zero residual mass everywhere) every rank switches to
      p_n, whose shard masses are A_r = e^{lse_r(n) - M} (exact identity);
  X3  the inverse CDF over ascending ids = the rank whose exclusive prefix
      interval of A holds T = u * sum A, then the local inverse CDF at
      (T - P_r) / e^{lse_r - M}; the tokens (-1 elsewhere) are gathered and
      every rank takes the maximum.

`gather(obj) -> list over ranks` and `allmax(np.ndarray) -> np.ndarray` are
injected (a plain loop in one process, or torch.distributed).
"""
from __future__ import annotations

import numpy as np

from .verify_np import bf16_to_f64


def shard_bounds(V: int, nranks: int):
    """128-row aligned contiguous split in rank order (nj_shard_range's rule)."""
    T = (V + 127) // 128
    return [(min(V, (T * r // nranks) * 128), min(V, (T * (r + 1) // nranks) * 128)) for r in range(nranks)]


def rank_step(rank, nranks, hidden_bits, W_bits, draft_tokens, draft_probs, gamma, uniforms, gather, allmax):
    H = bf16_to_f64(hidden_bits)
    W = bf16_to_f64(W_bits)
    V = W.shape[0]
    vb, ve = shard_bounds(V, nranks)[rank]
    L = H @ W[vb:ve].T                          # this rank's logits [N, V_r]
    gam = np.asarray(gamma, np.int64)
    B = gam.shape[0]
    ro = np.concatenate([[0], np.cumsum(gam + 1)])
    x_all = np.asarray(draft_tokens, np.int64).reshape(-1)
    q_all = np.asarray(draft_probs, np.float64)
    u = np.asarray(uniforms, np.float64).reshape(-1)

    def lse_of(v):
        m = v.max()
        return m + np.log(np.exp(v - m).sum())

    # ---- X1: per draft row (lse_r, owned draft logit)
    drows = [ro[b] + i for b in range(B) for i in range(gam[b])]
    x1 = np.array([[lse_of(L[j]), L[j, x - vb] if vb <= x < ve else np.nan]
                   for j, x in zip(drows, x_all)], np.float64).reshape(-1, 2)
    all1 = gather(x1)                           # list over ranks
    lse_d = np.array([lse_of(np.array([a[g, 0] for a in all1])) for g in range(len(drows))])
    dl = np.array([next(a[g, 1] for a in all1 if not np.isnan(a[g, 1])) for g in range(len(drows))])
    # acceptance (identical on every rank)
    n_out = np.zeros(B, np.int32)
    resid = np.zeros(B, bool)
    lse_used = np.zeros(B)
    g0 = 0
    for b in range(B):
        n = gam[b]
        for i in range(gam[b]):
            pd = np.exp(dl[g0 + i] - lse_d[g0 + i])
            if not (u[ro[b] + i] * q_all[g0 + i, x_all[g0 + i]] < pd):
                n = i
                break
        n_out[b] = n
        resid[b] = n < gam[b]
        if resid[b]:
            lse_used[b] = lse_d[g0 + n]
        g0 += gam[b]
    # ---- X2: local masses
    wloc, ploc = [], []
    x2 = np.zeros((B, 3))
    g0 = 0
    for b in range(B):
        row = L[ro[b] + n_out[b]]
        lr = lse_of(row)
        if resid[b]:
            w = np.maximum(np.exp(row - lse_used[b]) - q_all[g0 + n_out[b], vb:ve], 0.0)
            x2[b] = (lse_used[b], w.sum(), lr)
        else:
            w = np.exp(row - lr)
            x2[b] = (lr, w.sum(), lr)
        wloc.append(w)
        ploc.append(np.exp(row - lr))
        g0 += gam[b]
    all2 = gather(x2)
    # ---- X3: owner rank locates; tokens gathered, max over ranks taken locally
    tok = np.full(B, -1, np.int32)
    for b in range(B):
        lr = np.array([a[b, 0] for a in all2])
        Wr = np.array([a[b, 1] for a in all2])
        ln = np.array([a[b, 2] for a in all2])
        pos = Wr > 0
        if pos.any():
            M = lr[pos].max()
            A = np.where(pos, Wr * np.exp(lr - M), 0.0)
            ev, wl = np.exp(lr - M), wloc[b]
        else:                                   # R6 across shards: draw from p_n
            M = ln.max()
            A = np.exp(ln - M)
            ev, wl = A, ploc[b]
        T = u[ro[b] + gam[b]] * A.sum()
        P = np.concatenate([[0.0], np.cumsum(A)])
        own = [r for r in range(nranks) if A[r] > 0 and P[r] <= T < P[r + 1]]
        o = own[0] if own else int(np.nonzero(A > 0)[0][-1])
        if o != rank:
            continue
        c = np.cumsum(wl)
        t = int(np.searchsorted(c, (T - P[o]) / ev[o], side="right")) if own else len(c)
        if t >= len(c):
            t = int(np.nonzero(wl > 0)[0][-1])
        tok[b] = vb + t
    toks = gather(tok)
    return n_out, np.max(np.stack(toks), axis=0).astype(np.int32)
