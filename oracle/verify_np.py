"""Second, independent oracle: NumPy fp64 implementation of the same definition.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Written separately from
nj_oracle.c so that the two cross-check each other (SURVEY §8(c) "Second
oracle"): vectorised NumPy instead of C loops, np.searchsorted instead of a
running-sum scan, a different bf16 decoding route.  Small sizes only
(N <= 64, V <= 4096).

Definition followed (PAPER.md:23 Leviathan step, BJ steps 1-3, R2-R6):
  l = H W^T;  p_j = softmax(l_j);  accept draft i iff u_i q_i(x_i) < p_i(x_i);
  n = first failure else gamma;  w = max(0, p_n - q_n) if n < gamma else p_gamma;
  w = p_n if sum(w) == 0;  t = min{x : cumsum(w)[x] > u_gamma * sum(w)}.
"""
from __future__ import annotations

import numpy as np


def bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    """uint16 bf16 bit patterns -> float64 via the fp32 bit layout."""
    return (np.asarray(bits, np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def verify(hidden_bits, W_bits, draft_tokens, draft_probs, gamma, uniforms):
    H = bf16_to_f64(hidden_bits)
    W = bf16_to_f64(W_bits)
    V = W.shape[0]
    logits = H @ W.T                                   # step 1 (library matmul)
    m = logits.max(axis=1, keepdims=True)
    lse = (m + np.log(np.exp(logits - m).sum(axis=1, keepdims=True)))[:, 0]
    P = np.exp(logits - lse[:, None])                  # step 2
    q_all = np.asarray(draft_probs, np.float64)
    x_all = np.asarray(draft_tokens, np.int64).reshape(-1)
    u_all = np.asarray(uniforms, np.float64).reshape(-1)
    gam = np.asarray(gamma, np.int64)
    B = gam.shape[0]
    n_out = np.zeros(B, np.int32)
    t_out = np.zeros(B, np.int32)
    row = 0
    drf = 0
    for b in range(B):
        g = int(gam[b])
        n = g
        for i in range(g):                             # step 3: first rejection
            x = x_all[drf + i]
            if not (u_all[row + i] * q_all[drf + i, x] < P[row + i, x]):
                n = i
                break
        if n < g:                                      # residual
            w = np.maximum(P[row + n] - q_all[drf + n, :V], 0.0)
        else:                                          # bonus
            w = P[row + g].copy()
        if w.sum() == 0.0:
            w = P[row + n].copy()
        c = np.cumsum(w)
        T = u_all[row + g] * c[-1]
        t = int(np.searchsorted(c, T, side="right"))   # first index with c > T
        if t >= V:
            t = int(np.nonzero(w > 0)[0][-1])
        n_out[b] = n
        t_out[b] = t
        row += g + 1
        drf += g
    return {"accept_len": n_out, "next_token": t_out, "lse": lse, "P": P}
