"""Parity bookkeeping shared by the GPU tests: the CUDA path (through the C ABI)
against the fp64 oracle on identical inputs, with the near-tie rule of
BASELINE.json north_star / DESIGN.md R12.

  * Requests the oracle does not flag as ties: accept_len and next_token
    bit-exact.
  * Requests flagged NJ_FLAG_FALLBACK by the GPU (recomputed in fp64 by the
    certified fallback): bit-exact as well, unless an oracle margin is below
    1e-10 (fp64 summation order).
  * Excused requests (oracle margin within the 1e-6 band) are still checked:
    the GPU outcome must be one the method reaches when each tied decision
    goes either way -- the tied acceptance test flipped (u_i forced to 0 or 2),
    the draw moved to a token whose CDF interval meets [u - 1e-6, u + 1e-6].
    Those alternatives are computed by the oracle itself (verify_from_logits
    on the request's fp64 logits with the perturbed fp64 uniforms).
  * The number of excused requests must agree with the oracle's expected
    count sum_b p_tie(b) (Poisson-binomial; 4 sigma), so a broken tie
    classifier cannot make a test vacuous.
  * Counts are recorded in STATS and printed in pytest's terminal summary.

Test infrastructure only (imports oracle/).
"""
from __future__ import annotations

import math

import numpy as np

import oracle

STATS: list[dict] = []
EPS = oracle.TIE_EPS
GPU_FLAG_FALLBACK = 1


def _tested(n: int, g: int) -> range:
    return range(0, min(n, g - 1) + 1) if g > 0 else range(0)


def valid_outcomes(L, x, q, g: int, u, eps: float = EPS, start: int = 0, depth: int = 0) -> set:
    """All (accept_len, next_token) the definition yields when every decision
    within eps of its uniform may go either way (one request; L its fp64
    logits [g+1, V], x [g], q [g, V], u [g+1] fp64)."""
    u = np.asarray(u, np.float64).copy()
    r = oracle.verify_from_logits(L, x, q, np.array([g], np.int32), u, tie_eps=eps)
    n, t = int(r["accept_len"][0]), int(r["next_token"][0])
    if depth < 8:
        for i in _tested(n, g):
            if i >= start and abs(r["ratio"][i] - u[i]) <= eps:
                ua, ur = u.copy(), u.copy()
                ua[i], ur[i] = 0.0, 2.0        # forced accept (p > 0) / forced reject (a <= 2)
                return (valid_outcomes(L, x, q, g, ua, eps, i + 1, depth + 1) |
                        valid_outcomes(L, x, q, g, ur, eps, i + 1, depth + 1))
    out = {(n, t)}
    uf = u[g]
    lo, hi = float(r["F_lo"][0]), float(r["F_hi"][0])
    # walk to the neighbouring tokens whose interval meets [u - eps, u + eps]
    for _ in range(6):
        if not hi < uf + eps or hi >= 1.0:
            break
        u2 = u.copy()
        u2[g] = hi + 1e-10
        r2 = oracle.verify_from_logits(L, x, q, np.array([g], np.int32), u2, tie_eps=eps)
        out.add((n, int(r2["next_token"][0])))
        hi = float(r2["F_hi"][0])
    for _ in range(6):
        if not lo > uf - eps or lo <= 0.0:
            break
        u2 = u.copy()
        u2[g] = lo - 1e-10
        r2 = oracle.verify_from_logits(L, x, q, np.array([g], np.int32), u2, tie_eps=eps)
        out.add((n, int(r2["next_token"][0])))
        lo = float(r2["F_lo"][0])
    return out


def check(name, n, acc, nxt, r=None, gpu_flags=None, L=None, certified=False, gemm="c"):
    """Compare GPU outputs with the oracle for the batch `n` (Batch.to_numpy()).

    r: the oracle result if already computed (else computed here); L: the
    oracle's fp64 logits of all rows (computed on demand for excused
    requests); gpu_flags: the GPU's per-request NJ_FLAG_* bits (dbg.flags).
    Returns the oracle result."""
    g = np.asarray(n["gamma"], np.int32)
    B = g.shape[0]
    if r is None:
        if L is None:
            L = (oracle.logits_blas(n["hidden_bits"], n["W_bits"]) if gemm == "blas"
                 else oracle.logits(n["hidden_bits"], n["W_bits"]))
        r = oracle.verify_from_logits(L, n["draft_tokens"], n["draft_probs"], g, n["uniforms"])
    acc = np.asarray(acc)
    nxt = np.asarray(nxt)
    assert ((acc >= 0) & (acc <= g)).all(), "accept_len outside [0, gamma]"
    tie = r["tie"]
    fb = np.zeros(B, bool) if gpu_flags is None else (np.asarray(gpu_flags) & GPU_FLAG_FALLBACK) != 0
    tiny = (r["accept_margin"] < 1e-10) | (r["draw_margin"] < 1e-10)
    exact = ~tie | (fb & ~tiny)
    bad = np.nonzero(exact & ((acc != r["accept_len"]) | (nxt != r["next_token"])))[0]
    assert bad.size == 0, (name, "out-of-band mismatch", bad[:8], acc[bad[:8]], r["accept_len"][bad[:8]],
                           nxt[bad[:8]], r["next_token"][bad[:8]])
    # excused requests: the GPU outcome must be one of the tied branches
    ro = np.concatenate([[0], np.cumsum(g + 1)])
    do = np.concatenate([[0], np.cumsum(g)])
    excused = np.nonzero(~exact)[0]
    alt_used = 0
    u_all = np.asarray(n["uniforms"], np.float64)
    q_all = np.asarray(n["draft_probs"], np.float32)
    for b in excused:
        if acc[b] == r["accept_len"][b] and nxt[b] == r["next_token"][b]:
            continue
        Lb = (L[ro[b]:ro[b + 1]] if L is not None else
              oracle.logits(n["hidden_bits"][ro[b]:ro[b + 1]], n["W_bits"]))
        qb = q_all[do[b]:do[b + 1]] if g[b] else q_all[:1]
        outs = valid_outcomes(Lb, np.asarray(n["draft_tokens"][do[b]:do[b + 1]], np.int32), qb, int(g[b]),
                              u_all[ro[b]:ro[b + 1]])
        assert (int(acc[b]), int(nxt[b])) in outs, (name, "excused request outside its tie branches", int(b),
                                                     (int(acc[b]), int(nxt[b])), sorted(outs))
        alt_used += 1
    # the excused count against the oracle's expected tie count
    n_acc_tie = int(((r["flags"] & oracle.F_ACCEPT_TIE) != 0).sum())
    n_draw_tie = int(((r["flags"] & oracle.F_DRAW_TIE) != 0).sum())
    n_tie = int(tie.sum())
    expect = float(r["p_tie"].sum())
    sd = math.sqrt(max(expect, 1e-12))
    assert n_tie <= expect + 4 * sd + 3, (name, "more ties than expected", n_tie, expect)
    assert n_tie >= expect - 4 * sd - 3, (name, "fewer ties than expected", n_tie, expect)
    STATS.append({"test": name, "B": int(B), "N": int(g.sum() + B), "ties": n_tie, "accept_ties": n_acc_tie,
                  "draw_ties": n_draw_tie, "expected_ties": round(expect, 3), "excused": int(excused.size),
                  "excused_differing": alt_used, "fallback": int(fb.sum()), "certified": bool(certified)})
    return r
