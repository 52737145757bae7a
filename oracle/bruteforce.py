"""Exact cell-integration losslessness checker (V <= 8, gamma <= 3).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:23 states the verification "is lossless"; BJ asks to confirm "that
the emitted-token distribution equals the target distribution to 1e-12" by
brute-force enumeration on tiny vocabularies.  For fixed per-position target
rows p_0..p_gamma and draft rows q_0..q_{gamma-1} (R1), Leviathan's
guarantee is, for every k <= gamma, prefix a in V^k and token b:

    P(n >= k, y_{<k} = a, y_k = b) = prod_{i<k} min(p_i(a_i), q_i(a_i)) * p_k(b)   (*)

where y_k is the k-th emitted token (the accepted draft if n > k, the
resampled / bonus token if n = k).

Method.  Enumerate every draft tuple x in V^gamma (probability prod q_i(x_i)).
For each, the acceptance uniforms split into cells [0, min(1,a_i)) and
[min(1,a_i), 1) with a_i = p_i(x_i)/q_i(x_i); the final uniform splits at the
normalised CDF breakpoints of the residual / bonus row.  Cell boundaries come
from a closed-form NumPy computation of p (library matmul + softmax), NOT from
the implementation under test, which is evaluated once at each cell midpoint;
its outputs weighted by cell measure give its exact emitted law, compared
with (*).  Zero-width cells are skipped.
"""
from __future__ import annotations

import itertools

import numpy as np

from . import verify as _oracle_verify
from .verify_np import bf16_to_f64


def closed_form_p(hidden_bits, W_bits):
    l = bf16_to_f64(hidden_bits) @ bf16_to_f64(W_bits).T
    e = np.exp(l - l.max(axis=1, keepdims=True))
    return e / e.sum(axis=1, keepdims=True)


def build_cells(P, Q, gamma, f32_uniforms=False):
    """Enumerate cells.  P [gamma+1, V] closed-form target rows, Q [gamma, V]
    draft rows (fp64 copies of the fp32 inputs).  Returns a list of
    (x tuple, n, t, measure, uniforms[gamma+1])."""
    V = P.shape[1]
    cells = []
    for x in itertools.product(range(V), repeat=gamma):
        wx = 1.0
        for i, xi in enumerate(x):
            wx *= Q[i, xi]
        if wx == 0.0:
            continue
        acc = [min(1.0, P[i, xi] / Q[i, xi]) for i, xi in enumerate(x)]
        for n in range(gamma + 1):
            meas = wx
            u = np.zeros(gamma + 1)
            for i in range(n):
                meas *= acc[i]
                u[i] = acc[i] / 2.0
            if n < gamma:
                meas *= 1.0 - acc[n]
                u[n] = (acc[n] + 1.0) / 2.0
                w = np.maximum(P[n] - Q[n], 0.0)
                if w.sum() == 0.0:
                    w = P[n].copy()
            else:
                w = P[gamma].copy()
            if meas == 0.0:
                continue
            F = np.cumsum(w) / w.sum()
            lo = 0.0
            for t in range(V):
                hi = F[t] if t < V - 1 else 1.0
                if hi > lo and w[t] > 0:
                    uu = u.copy()
                    uu[gamma] = (lo + hi) / 2.0
                    if f32_uniforms:
                        uu = uu.astype(np.float32).astype(np.float64)
                    cells.append((x, n, t, meas * (hi - lo), uu))
                lo = hi
    return cells


def batch_inputs(hidden_bits, q_rows, cells, gamma):
    """Pack one request per cell (same gamma+1 hidden rows for every request)."""
    B = len(cells)
    H = np.tile(np.asarray(hidden_bits, np.uint16), (B, 1))
    x = np.array([c[0] for c in cells], np.int32).reshape(-1)
    Q = np.tile(np.asarray(q_rows, np.float32), (B, 1))
    u = np.concatenate([c[4] for c in cells])
    return H, x, Q, np.full(B, gamma, np.int32), u


def emitted_law(cells, n_out, t_out, V, gamma):
    """Weighted law of the implementation's outputs: hist[k][prefix..., b]."""
    hist = [np.zeros((V,) * (k + 1)) for k in range(gamma + 1)]
    for (x, _n, _t, meas, _u), n, t in zip(cells, n_out, t_out):
        for k in range(int(n) + 1):
            yk = x[k] if k < n else int(t)
            hist[k][tuple(x[:k]) + (yk,)] += meas
    return hist


def expected_law(P, Q, gamma):
    """Right-hand side of (*)."""
    V = P.shape[1]
    M = np.minimum(P[:gamma], Q)
    out = []
    for k in range(gamma + 1):
        h = np.zeros((V,) * (k + 1))
        for a in itertools.product(range(V), repeat=k):
            pr = 1.0
            for i, ai in enumerate(a):
                pr *= M[i, ai]
            h[a] = pr * P[k]
        out.append(h)
    return out


def check(hidden_bits, W_bits, q_rows, gamma, impl=None):
    """Run the brute force.  ``impl(H, W, x, Q, gammas, u) -> (n, t)`` defaults
    to the C oracle.  Returns (max abs error of (*), E[n], closed-form E[n],
    total mass, cell-label mismatches)."""
    P = closed_form_p(hidden_bits, W_bits)
    Qd = np.asarray(q_rows, np.float32).astype(np.float64)
    V = P.shape[1]
    cells = build_cells(P, Qd, gamma)
    H, x, Q, g, u = batch_inputs(hidden_bits, q_rows, cells, gamma)
    if impl is None:
        r = _oracle_verify(H, W_bits, x, Q, g, u)
        n_out, t_out = r["accept_len"], r["next_token"]
    else:
        n_out, t_out = impl(H, W_bits, x, Q, g, u)
    mism = sum(1 for c, n, t in zip(cells, n_out, t_out) if (c[1], c[2]) != (int(n), int(t)))
    got = emitted_law(cells, n_out, t_out, V, gamma)
    exp_ = expected_law(P, Qd, gamma)
    err = max(float(np.abs(a - b).max()) for a, b in zip(got, exp_))
    total = float(sum(c[3] for c in cells))
    En = float(sum(c[3] * int(n) for c, n in zip(cells, n_out)))
    beta = np.minimum(P[:gamma], Qd).sum(axis=1)
    En_cf = float(sum(np.prod(beta[:k]) for k in range(1, gamma + 1)))
    return {"max_err": err, "E_n": En, "E_n_closed_form": En_cf, "total": total,
            "label_mismatches": mism, "n_cells": len(cells)}
