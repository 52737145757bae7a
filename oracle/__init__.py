"""fp64 CPU oracle for batched speculative-decoding verification.

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with the CUDA path (``paper_2512_22420_b200``)
and neither imports the other; the only common module is the seeded input
generator ``synth.inputs``, which holds none of the method's arithmetic.

Contents
  nj_oracle.c     plain C fp64 oracle (GEMM, softmax, Leviathan rejection
                  sampling with supplied uniforms) -- PAPER.md:23, BJ steps 1-3.
  verify_np.py    an independent NumPy fp64 implementation of the same
                  definition (second oracle; small sizes only).
  bruteforce.py   exact cell-integration losslessness checker (V <= 8).
  bandit_ref.py   plain-Python Algorithm 1 / Eq. 3 reference.

Every function here is pinned by ``tests/test_oracle_pins.py`` /
``tests/test_bandit.py`` against facts the paper and the mathematics fix;
the only unpinned quantities are the path's throughput and the realised
acceptance rate of the synthetic draft.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nj_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

TIE_EPS = 1e-6  # DESIGN.md R12: near-tie band of BJ ("within 1e-6 of the uniform")

# oracle_debug flag bits (mirror of nj_oracle.c; oracle-internal)
F_ACCEPT_TIE, F_DRAW_TIE, F_ZERO_MASS, F_CLAMP, F_Q_ZERO = 1, 2, 4, 8, 16


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no -ffast-math; summation order is part
    of the definition)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp.%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I64, I32, D = ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        lib.oracle_logits.argtypes = [P, P, I64, P, I64, I64, P, ctypes.c_int]
        lib.oracle_logits.restype = ctypes.c_int
        lib.oracle_verify.argtypes = [P, P, I64, I64, P, P, I64, P, P, I32, P, P,
                                      P, P, P, P, P, P, P, P, P, P, D, ctypes.c_int]
        lib.oracle_verify.restype = ctypes.c_int
        lib.oracle_verify_logits.argtypes = [P, I64, P, P, I64, P, P, I32, P, P,
                                             P, P, P, P, P, P, P, P, P, P, D, ctypes.c_int]
        lib.oracle_verify_logits.restype = ctypes.c_int
        lib.oracle_sample_from_logits.argtypes = [P, I64, I64, P, P, I64, P, I32, P, P,
                                                  P, P, P, D, ctypes.c_int]
        lib.oracle_sample_from_logits.restype = ctypes.c_int
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def bf16_bits(a) -> np.ndarray:
    """Accept a uint16 bit array (or torch bf16 tensor) and return uint16 bits."""
    if hasattr(a, "view") and hasattr(a, "dtype") and str(a.dtype) == "torch.bfloat16":
        import torch
        return a.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)
    a = np.asarray(a)
    assert a.dtype == np.uint16, a.dtype
    return a


def logits(hidden_bits, W_bits, rows=None, nthreads: int = 0) -> np.ndarray:
    """fp64 logits l[r, x] = sum_k W[x,k] h[rows[r],k] (P:23 step 1)."""
    H = _c(bf16_bits(hidden_bits), np.uint16)
    Wb = _c(bf16_bits(W_bits), np.uint16)
    V, d = Wb.shape
    r = None if rows is None else _c(rows, np.int32)
    n = H.shape[0] if r is None else r.shape[0]
    out = np.empty((n, V), np.float64)
    if _load().oracle_logits(_ptr(H), _ptr(r), n, _ptr(Wb), V, d, _ptr(out), nthreads):
        raise MemoryError("oracle_logits failed")
    return out


def weight_f64(W_bits) -> np.ndarray:
    """bf16 bits -> fp64 (exact), for reuse across logits_blas calls."""
    Wb = _c(bf16_bits(W_bits), np.uint16)
    return (Wb.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def logits_blas(hidden_bits, W_bits, rows=None, v_chunk: int = 16384, W64=None) -> np.ndarray:
    """Step 1 with a library matmul (numpy/BLAS fp64) instead of the C loops:
    the same definition l[r, x] = sum_k W[x,k] h[r,k] of the identical bf16
    values, summed in the library's order (pinned against oracle.logits to
    1e-12 relative, tests/test_oracle_pins.py).  Used only where the C loops
    would take minutes (full-size batches of >= 1000 rows)."""
    H = _c(bf16_bits(hidden_bits), np.uint16)
    if rows is not None:
        H = H[np.asarray(rows, np.int64)]
    h = (H.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    if W64 is not None:
        return h @ W64.T
    Wb = _c(bf16_bits(W_bits), np.uint16)
    V = Wb.shape[0]
    out = np.empty((h.shape[0], V), np.float64)
    for v0 in range(0, V, v_chunk):
        w = (Wb[v0:v0 + v_chunk].astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        np.matmul(h, w.T, out=out[:, v0:v0 + w.shape[0]])
    return out


def verify(hidden_bits, W_bits, draft_tokens, draft_probs, gamma, uniforms,
           tie_eps: float = TIE_EPS, nthreads: int = 0, gemm: str = "c", temperature: float = 1.0) -> dict:
    """Full fp64 verification of a packed ragged batch (layout of include/nj.h).

    ``uniforms`` may be fp32 (converted exactly) or fp64 (brute force, tie
    branches).  ``gemm``: "c" (the plain loops of nj_oracle.c) or "blas"
    (logits_blas).  Returns dict with accept_len, next_token and the fp64
    debug arrays (see verify_from_logits)."""
    H = _c(bf16_bits(hidden_bits), np.uint16)
    Wb = _c(bf16_bits(W_bits), np.uint16)
    V, d = Wb.shape
    g = _c(gamma, np.int32)
    N = int(g.sum()) + g.shape[0]
    assert H.shape == (N, d), (H.shape, N, d)
    L = logits_blas(H, Wb) if gemm == "blas" else logits(H, Wb, nthreads=nthreads)
    if temperature != 1.0:
        # target at temperature T (R17): p = softmax(l / T)
        L = L / float(temperature)
    return verify_from_logits(L, draft_tokens, draft_probs, gamma, uniforms, tie_eps=tie_eps, nthreads=nthreads)


def verify_from_logits(L, draft_tokens, draft_probs, gamma, uniforms, tie_eps: float = TIE_EPS,
                       nthreads: int = 0) -> dict:
    """Steps 2-6 of the verification given the fp64 logits L [N, V] of the
    packed rows (step 1).  Returns accept_len, next_token and the fp64 debug
    arrays: lse [N], p_draft / ratio [G] (a_i = p_i(x_i)/q_i(x_i)), mass [B]
    (W_b), F_lo / F_hi [B] (the drawn token's normalised CDF interval), flags,
    accept_margin / draw_margin [B], p_tie [B] (probability over the
    uniforms that the request is flagged a tie, R12) and tie."""
    L = _c(L, np.float64)
    N, V = L.shape
    g = _c(gamma, np.int32)
    B = g.shape[0]
    G = int(g.sum())
    assert N == G + B, (N, G, B)
    x = _c(draft_tokens, np.int32).reshape(-1)
    assert x.shape[0] == G
    q = np.asarray(draft_probs, dtype=np.float32)
    if G == 0:
        q = np.zeros((1, V), np.float32)
    q = np.ascontiguousarray(q.reshape(max(G, 1), -1))
    ldq = q.shape[1]
    assert ldq >= V
    u = _c(np.asarray(uniforms, dtype=np.float64), np.float64).reshape(-1)
    assert u.shape[0] == N
    out = {
        "accept_len": np.empty(B, np.int32), "next_token": np.empty(B, np.int32),
        "lse": np.empty(N), "p_draft": np.empty(max(G, 1)), "ratio": np.empty(max(G, 1)),
        "mass": np.empty(B), "F_lo": np.empty(B), "F_hi": np.empty(B),
        "flags": np.empty(B, np.int32), "accept_margin": np.empty(B), "draw_margin": np.empty(B),
        "p_tie": np.empty(B),
    }
    xs = x if G else np.zeros(1, np.int32)
    rc = _load().oracle_verify_logits(
        _ptr(L), V, _ptr(xs), _ptr(q), ldq, _ptr(g), _ptr(u), B,
        _ptr(out["accept_len"]), _ptr(out["next_token"]), _ptr(out["lse"]),
        _ptr(out["p_draft"]), _ptr(out["ratio"]), _ptr(out["mass"]), _ptr(out["F_lo"]),
        _ptr(out["F_hi"]), _ptr(out["flags"]), _ptr(out["accept_margin"]),
        _ptr(out["draw_margin"]), _ptr(out["p_tie"]), tie_eps, nthreads)
    if rc:
        raise MemoryError("oracle_verify_logits failed")
    out["p_draft"] = out["p_draft"][:G]
    out["ratio"] = out["ratio"][:G]
    out["tie"] = (out["flags"] & (F_ACCEPT_TIE | F_DRAW_TIE)) != 0
    return out


def verify_greedy(hidden_bits, W_bits, draft_tokens, gamma, tie_gap: float = 1e-4, nthreads: int = 0) -> dict:
    """Verification against the argmax target (the
    temperature -> 0 limit of PAPER.md:23's sampled verification): a_j =
    argmax_x l_j(x) in fp64 (ties -> lowest id); request b accepts its drafts
    up to the first x_i != a_i and emits a_n.  ``tie`` marks requests whose
    decision consulted a row with top-2 logit gap <= tie_gap (where fp32
    logits may order the top two differently)."""
    L = logits(hidden_bits, W_bits, nthreads=nthreads)
    a = L.argmax(axis=1)
    top2 = np.sort(L, axis=1)[:, -2:] if L.shape[1] > 1 else np.concatenate([L - np.inf, L], axis=1)
    gap = top2[:, 1] - top2[:, 0]
    g = np.asarray(gamma, np.int64)
    x = np.asarray(draft_tokens, np.int64).reshape(-1)
    B = g.shape[0]
    acc = np.empty(B, np.int32)
    nxt = np.empty(B, np.int32)
    tie = np.zeros(B, bool)
    ro = 0
    for b in range(B):
        g0 = ro - b
        n = int(g[b])
        for i in range(int(g[b])):
            if x[g0 + i] != a[ro + i]:
                n = i
                break
        acc[b], nxt[b] = n, a[ro + n]
        tie[b] = bool((gap[ro:ro + n + 1] <= tie_gap).any())
        ro += int(g[b]) + 1
    return {"accept_len": acc, "next_token": nxt, "argmax": a, "gap": gap, "tie": tie}


def propose(hidden_bits, W_bits, uniforms, tie_eps: float = TIE_EPS, nthreads: int = 0,
            temperature: float = 1.0) -> dict:
    """Draft-side proposal step (the
    draft proposes x ~ q): q_b = softmax(l_b) of the draft LM head and x_b the
    inverse-CDF draw of q_b with uniform u_b.  Written as the definition's two
    pinned pieces: the fp64 logits (step 1) and verification with gamma = 0,
    which draws from p_0 = softmax(l_0) (test_gamma0_is_inverse_cdf_of_p).
    Returns tokens, q (fp64 [B, V]), lse and the draw's tie mask."""
    L = logits(hidden_bits, W_bits, nthreads=nthreads) / float(temperature)
    B, V = L.shape
    r = verify_from_logits(L, np.zeros(0, np.int32), np.zeros((0, V), np.float32), np.zeros(B, np.int32),
                           uniforms, tie_eps=tie_eps, nthreads=nthreads)
    q = np.exp(L - r["lse"][:, None])
    return {"tokens": r["next_token"], "q": q, "lse": r["lse"], "tie": r["tie"]}


def sample_from_logits(logits32, residual, q, u, tie_eps: float = TIE_EPS,
                       nthreads: int = 0) -> dict:
    """Stage-isolated sampler oracle on fp32 logits (R11(ii))."""
    L = _c(logits32, np.float32)
    B, V = L.shape
    res = _c(residual, np.int32)
    qq = _c(q, np.float32).reshape(B, -1)
    uu = _c(np.asarray(u, np.float64), np.float64)
    out = {"next_token": np.empty(B, np.int32), "mass": np.empty(B), "F_lo": np.empty(B),
           "F_hi": np.empty(B), "flags": np.empty(B, np.int32)}
    rc = _load().oracle_sample_from_logits(
        _ptr(L), V, V, _ptr(res), _ptr(qq), qq.shape[1], _ptr(uu), B,
        _ptr(out["next_token"]), _ptr(out["mass"]), _ptr(out["F_lo"]), _ptr(out["F_hi"]),
        _ptr(out["flags"]), tie_eps, nthreads)
    if rc:
        raise MemoryError("oracle_sample_from_logits failed")
    out["tie"] = (out["flags"] & F_DRAW_TIE) != 0
    return out
