"""Pins of the fp64 oracle (oracle/) against facts fixed by the paper and the
mathematics -- none of them re-types the oracle's own formula:

  GEMM          numpy float64 matmul of the identical values (library routine)
  softmax       scipy.special.logsumexp; sum p = 1 (closed form)
  gamma = 0     searchsorted(cumsum(p), u * sum p, 'right')  (textbook inverse CDF)
  q = p         every draft accepted for u < 1 (special case)
  p one-hot     any x != y rejected, draw = y   (special case)
  q one-hot     accept iff u < p(x)            (special case)
  forced u      u = 0 accepts, u = 1 - 2^-24 rejects unless a > u (special case)
  lossless      brute-force cell integration, V <= 8, gamma <= 3, to 1e-12
                ("lossless"; BJ)
  E[n]          sum_k prod_{i<k} beta_i, beta_i = sum_x min(p_i, q_i) (closed form)
  geometric     identical rows: E[n+1] = (1 - beta^(g+1)) / (1 - beta)
  invariants    0 <= n <= gamma; w(t) > 0; residual draws have p(t) > q(t)
  2nd oracle    an independent NumPy implementation agrees (decisions exact)
"""
import numpy as np
import pytest
import scipy.special

import oracle
from oracle import bruteforce
from oracle.verify_np import bf16_to_f64
from oracle.verify_np import verify as np_verify
from synth.inputs import dyadic_rows, make_batch


def _np(b):
    return b.to_numpy()


def _verify(n, **kw):
    return oracle.verify(n["hidden_bits"], n["W_bits"], n["draft_tokens"], n["draft_probs"], n["gamma"],
                         n["uniforms"], **kw)


def _exact_p(n):
    l = bf16_to_f64(n["hidden_bits"]) @ bf16_to_f64(n["W_bits"]).T
    return scipy.special.softmax(l, axis=1), l


def _bf16(x):
    x = np.asarray(x, np.float32)
    return (x.view(np.uint32) >> 16).astype(np.uint16)   # exact for bf16-representable values


# ------------------------------------------------------------------ GEMM, softmax
@pytest.mark.parametrize("V,d,R", [(32, 16, 4), (1000, 64, 7), (4096, 256, 3)])
def test_gemm_matches_numpy(V, d, R):
    b = make_batch(R, 0, V=V, d=d, seed=V + d)
    n = _np(b)
    got = oracle.logits(n["hidden_bits"], n["W_bits"])
    ref = bf16_to_f64(n["hidden_bits"]) @ bf16_to_f64(n["W_bits"]).T
    assert np.max(np.abs(got - ref) / (np.abs(ref) + 1e-300)) < 1e-12


def test_softmax_closed_form():
    b = make_batch(6, 2, V=3000, d=64, seed=3)
    n = _np(b)
    r = _verify(n)
    P, l = _exact_p(n)
    np.testing.assert_allclose(r["lse"], scipy.special.logsumexp(l, axis=1), rtol=0, atol=1e-12)
    np.testing.assert_allclose(P.sum(1), 1.0, atol=1e-12)


def test_second_oracle_agrees():
    for seed in range(5):
        b = make_batch(9, "mixed:5", V=777, d=32, seed=seed)
        n = _np(b)
        r = _verify(n)
        r2 = np_verify(n["hidden_bits"], n["W_bits"], n["draft_tokens"], n["draft_probs"], n["gamma"], n["uniforms"])
        assert (r["accept_len"] == r2["accept_len"]).all()
        assert (r["next_token"] == r2["next_token"]).all()
        np.testing.assert_allclose(r["lse"], r2["lse"], atol=1e-12)


# ------------------------------------------------------------------ special cases
def test_gamma0_is_inverse_cdf_of_p():
    b = make_batch(40, 0, V=500, d=32, seed=11)
    n = _np(b)
    r = _verify(n)
    P, _ = _exact_p(n)
    assert (r["accept_len"] == 0).all()
    for i in range(40):
        c = np.cumsum(P[i])
        t = int(np.searchsorted(c, float(n["uniforms"][i]) * c[-1], side="right"))
        if r["tie"][i]:
            continue
        assert r["next_token"][i] == t


def test_q_equals_p_accepts_everything():
    b = make_batch(12, 3, V=300, d=32, seed=5)
    n = _np(b)
    P, _ = _exact_p(n)
    g = n["gamma"]
    rows = np.concatenate([np.arange(o, o + gg) for o, gg in zip(np.concatenate([[0], np.cumsum(g + 1)[:-1]]), g)])
    n["draft_probs"] = P[rows].astype(np.float32)
    n["uniforms"] = np.minimum(n["uniforms"], np.float32(0.999))   # a = p/q = 1 -/+ 6e-8 (fp32 q)
    r = _verify(n)
    assert (r["accept_len"] == g).all()


def test_p_one_hot_draws_its_token():
    """W row y dominates by > 745 nats so p(x != y) underflows to exactly 0."""
    V, d = 16, 16
    rng = np.random.default_rng(0)
    W = rng.standard_normal((V, d)).astype(np.float32) * 0.01
    y = 11
    W[y] = 64.0                      # l_y = 64 * sum(h) = 1024 with h = 1
    H = np.ones((4, d), np.float32)  # gamma = 3 -> 4 rows
    q = dyadic_rows(np.full((3, V), 1.0 / V))
    x = np.array([3, 5, 7], np.int32)
    for u in [0.0, 0.3, 0.999]:
        r = oracle.verify(_bf16(H), _bf16(W), x, q, np.array([3], np.int32), np.array([u, u, u, u]))
        assert r["accept_len"][0] == 0 and r["next_token"][0] == y
    # drafting y itself is always accepted (a = 1/q > 1)
    r = oracle.verify(_bf16(H), _bf16(W), np.array([y, y, y], np.int32), q, np.array([3], np.int32),
                      np.array([0.9, 0.9, 0.9, 0.5]))
    assert r["accept_len"][0] == 3 and r["next_token"][0] == y


def test_q_one_hot_accepts_iff_u_below_p():
    b = make_batch(1, 1, V=64, d=16, seed=2)
    n = _np(b)
    P, _ = _exact_p(n)
    x = int(np.argmax(P[0]))
    q = np.zeros((1, 64), np.float32)
    q[0, x] = 1.0
    n["draft_probs"], n["draft_tokens"] = q, np.array([x], np.int32)
    px = P[0, x]
    for u, acc in [(px * 0.999, 1), (px * 1.001, 0), (0.0, 1)]:
        n["uniforms"] = np.array([u, 0.5])
        r = _verify(n)
        assert r["accept_len"][0] == acc


def test_forced_branches():
    """u_i = 0 always accepts a token with p > 0; u_i = 1 - 2^-24 rejects unless a_i > u_i."""
    b = make_batch(1, 3, V=32, d=16, seed=4)
    n = _np(b)
    top = np.float32(1.0 - 2.0 ** -24)
    for k in range(4):   # accept k drafts, then reject (or accept all when k = 3)
        u = np.array([0.0] * k + [top] * (3 - k) + [0.5])
        r = _verify({**n, "uniforms": u})
        a = r["ratio"]
        expect = k
        while expect < 3 and a[expect] > top:   # a draft with a > 1 - 2^-24 is accepted anyway
            expect += 1
        assert r["accept_len"][0] == expect


# ------------------------------------------------------------------ losslessness
@pytest.mark.parametrize("V,gamma,seed", [(6, 3, 0), (8, 3, 1), (8, 2, 2), (5, 1, 3), (8, 1, 4), (7, 0, 5),
                                          (4, 3, 6)])
def test_losslessness_bruteforce(V, gamma, seed):
    b = make_batch(1, gamma, V=V, d=16, seed=seed)
    n = _np(b)
    q = dyadic_rows(n["draft_probs"]) if gamma else n["draft_probs"]
    r = bruteforce.check(n["hidden_bits"], n["W_bits"], q, gamma)
    assert r["label_mismatches"] == 0
    assert abs(r["total"] - 1.0) < 1e-12
    assert r["max_err"] < 1e-12
    assert abs(r["E_n"] - r["E_n_closed_form"]) < 1e-12


def test_losslessness_with_zero_q_entries():
    """Drafts never propose q = 0 tokens; residual mass comes from them (R7/R8)."""
    b = make_batch(1, 2, V=8, d=16, seed=9)
    n = _np(b)
    q = np.asarray(n["draft_probs"], np.float64)
    q[:, [1, 6]] = 0.0
    q = dyadic_rows(q, min_count=0)
    q[:, [1, 6]] = 0.0
    q = dyadic_rows(q, min_count=0)
    r = bruteforce.check(n["hidden_bits"], n["W_bits"], q, 2)
    assert r["label_mismatches"] == 0 and r["max_err"] < 1e-12


def test_identical_rows_geometric_expectation():
    """Identical p and q at every position: n+1 is truncated-geometric with
    E[n+1] = (1 - beta^(g+1)) / (1 - beta) (Leviathan Eq. 1)."""
    V, d, g = 8, 16, 3
    b = make_batch(1, g, V=V, d=d, seed=12)
    n = _np(b)
    H = np.tile(n["hidden_bits"][:1], (g + 1, 1))
    q = dyadic_rows(np.tile(n["draft_probs"][:1], (g, 1)))
    r = bruteforce.check(H, n["W_bits"], q, g)
    P = bruteforce.closed_form_p(H[:1], n["W_bits"])[0]
    beta = np.minimum(P, q[0].astype(np.float64)).sum()
    assert abs((r["E_n"] + 1.0) - (1 - beta ** (g + 1)) / (1 - beta)) < 1e-12


# ------------------------------------------------------------------ invariants
def test_invariants_random():
    for seed in range(4):
        b = make_batch(30, "mixed:5", V=2000, d=32, seed=seed, q_vocab=1900)
        n = _np(b)
        r = _verify(n)
        P, _ = _exact_p(n)
        g = n["gamma"]
        ro = np.concatenate([[0], np.cumsum(g + 1)[:-1]])
        do = np.concatenate([[0], np.cumsum(g)[:-1]])
        assert ((0 <= r["accept_len"]) & (r["accept_len"] <= g)).all()
        for b_ in range(len(g)):
            nb, t = r["accept_len"][b_], r["next_token"][b_]
            p = P[ro[b_] + nb]
            if nb < g[b_]:
                q = n["draft_probs"][do[b_] + nb].astype(np.float64)
                assert p[t] > q[t]                      # residual draw has positive weight
            else:
                assert p[t] > 0


def test_zero_residual_mass_draws_from_p():
    """R6: if max(0, p_n - q_n) sums to 0, draw from p_n."""
    b = make_batch(1, 1, V=16, d=16, seed=3)
    n = _np(b)
    P, _ = _exact_p(n)
    # q_0 = p_0 rounded up to fp32 so that p - q <= 0 everywhere
    q = np.nextafter(P[0].astype(np.float32), np.float32(2.0)).reshape(1, -1)
    x = int(np.argmin(P[0]))
    n = {**n, "draft_probs": q, "draft_tokens": np.array([x], np.int32),
         "uniforms": np.array([1.0 - 1e-12, 0.37])}
    r = _verify(n)
    assert r["accept_len"][0] == 0
    assert r["flags"][0] & oracle.F_ZERO_MASS
    c = np.cumsum(P[0])
    assert r["next_token"][0] == int(np.searchsorted(c, 0.37 * c[-1], side="right"))


# ------------------------------------------------------------------ golden C1
def test_golden_c1_fixture():
    """BJ config 1 (B=1, gamma=3, V=32, d=16) with fixed uniforms; fixture
    written by scripts/make_golden.py (calls only oracle/)."""
    import json
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "c1_fixed_uniforms.json")
    g = json.load(open(path))
    b = make_batch(1, 3, V=32, d=16, seed=g["seed"])
    n = _np(b)
    for case in g["cases"]:
        r = _verify({**n, "uniforms": np.array(case["uniforms"], np.float32)})
        assert int(r["accept_len"][0]) == case["accept_len"]
        assert int(r["next_token"][0]) == case["next_token"]


# ------------------------------------------------------------------ stage oracle
def test_sample_from_logits_matches_definition():
    rng = np.random.default_rng(7)
    B, V = 6, 400
    L = (rng.standard_normal((B, V)) * 3).astype(np.float32)
    q = scipy.special.softmax(0.9 * (L + rng.standard_normal((B, V))), axis=1).astype(np.float32)
    res = np.array([1, 0, 1, 1, 0, 1], np.int32)
    u = rng.integers(0, 1 << 24, size=B) * 2.0 ** -24
    r = oracle.sample_from_logits(L, res, q, u)
    for b in range(B):
        p = scipy.special.softmax(L[b].astype(np.float64))
        w = np.maximum(p - q[b], 0) if res[b] else p
        c = np.cumsum(w)
        t = int(np.searchsorted(c, u[b] * c[-1], side="right"))
        assert abs(r["mass"][b] - w.sum()) < 1e-12
        if not r["tie"][b]:
            assert r["next_token"][b] == t


def test_propose_draws_from_softmax_and_q_sums_to_one():
    """oracle.propose (draft proposal): q rows are
    probability vectors (sum 1 to 1e-12), equal to the fp64 softmax of the
    logits, and the token is the inverse-CDF draw of q -- checked with
    np.searchsorted on the cumulative q (an independent routine); a one-hot
    logit row (one huge logit) draws its token for every u."""
    b = make_batch(24, 0, V=700, d=32, seed=5)
    n = _np(b)
    r = oracle.propose(n["hidden_bits"], n["W_bits"], n["uniforms"])
    assert np.allclose(r["q"].sum(axis=1), 1.0, atol=1e-12, rtol=0)
    for i in range(24):
        c = np.cumsum(r["q"][i])
        t = int(np.searchsorted(c, float(n["uniforms"][i]) * c[-1], side="right"))
        if not r["tie"][i]:
            assert r["tokens"][i] == t
    # peaked row: a hidden state aligned with one W row dominates
    W = np.zeros((16, 8), np.float32); W[np.arange(16), np.arange(16) % 8] = 0.01
    W[11] = 0.0; W[11, 3] = 64.0
    h = np.zeros((3, 8), np.float32); h[:, 3] = 4.0
    u = np.array([0.25, 0.5, 0.999], np.float32)
    import torch
    bf = lambda a: torch.tensor(a, dtype=torch.bfloat16)
    rp = oracle.propose(bf(h), bf(W), u)
    assert (rp["tokens"] == 11).all()


def test_greedy_is_zero_temperature_limit():
    """oracle.verify_greedy equals the (pinned) sampled verification of the same
    batch with W scaled by 2^16 -- exact in bf16 and in the fp64 logits, so the
    target softmax is one-hot to < e^-6 wherever the top-2 gap exceeds 1e-4
    (the greedy tie band)."""
    import torch
    b = make_batch(30, "mixed:5", V=300, d=32, seed=13)
    n = _np(b)
    Ws = (b.W.float() * 65536.0).to(torch.bfloat16)
    assert torch.equal(Ws.float(), b.W.float() * 65536.0)
    r_s = oracle.verify(n["hidden_bits"], oracle.bf16_bits(Ws), n["draft_tokens"], n["draft_probs"], n["gamma"],
                        n["uniforms"])
    r_g = oracle.verify_greedy(n["hidden_bits"], n["W_bits"], n["draft_tokens"], n["gamma"])
    ok = ~r_g["tie"]
    assert ok.sum() >= 25
    assert (r_s["accept_len"][ok] == r_g["accept_len"][ok]).all()
    assert (r_s["next_token"][ok] == r_g["next_token"][ok]).all()
    # and a draft that copies the argmax is accepted in full
    L = oracle.logits(n["hidden_bits"], n["W_bits"])
    g = n["gamma"]
    ro = np.concatenate([[0], np.cumsum(g + 1)])
    x = np.concatenate([L[ro[b]:ro[b] + g[b]].argmax(axis=1) for b in range(len(g))]).astype(np.int32)
    r2 = oracle.verify_greedy(n["hidden_bits"], n["W_bits"], x, g)
    assert (r2["accept_len"] == g).all()
