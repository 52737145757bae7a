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


# ------------------------------------------------------------------ tie classifier (R12)
def _one_row_case(V=64, d=16, seed=21):
    b = make_batch(1, 0, V=V, d=d, seed=seed)
    n = _np(b)
    P, _ = _exact_p(n)
    return n, P[0]


def test_tie_classifier_draw_band():
    """Draw tie iff |u - F(t)| or |u - F(t-1)| <= 1e-6, F = cumsum(p) / sum(p)
    computed here with np.cumsum of the scipy softmax: u = F(k) -/+ 5e-7 is a
    tie (tokens k / k+1), u = F(k) -/+ 2e-6 is not; F_lo / F_hi / draw_margin
    are the interval ends and the distance to the nearer one."""
    n, p = _one_row_case()
    F = np.cumsum(p) / p.sum()
    widths = np.diff(np.concatenate([[0.0], F]))
    ks = [k for k in range(len(p) - 1) if widths[k] > 1e-5 and widths[k + 1] > 1e-5][:6]
    assert len(ks) >= 3
    for k in ks:
        for delta, tie in [(-2e-6, False), (-5e-7, True), (5e-7, True), (2e-6, False)]:
            u = np.array([F[k] + delta])
            r = oracle.verify(n["hidden_bits"], n["W_bits"], np.zeros(0, np.int32), np.zeros((0, 64), np.float32),
                              np.array([0], np.int32), u)
            t = k if delta < 0 else k + 1
            assert r["next_token"][0] == t
            assert bool(r["flags"][0] & oracle.F_DRAW_TIE) == tie, (k, delta)
            assert bool(r["tie"][0]) == tie
            assert abs(r["F_lo"][0] - (F[t - 1] if t else 0.0)) < 1e-12 and abs(r["F_hi"][0] - F[t]) < 1e-12
            assert abs(r["draw_margin"][0] - abs(delta)) < 1e-12


def test_tie_classifier_accept_band():
    """Acceptance tie iff |a_i - u_i| <= 1e-6 for a TESTED draft, a_i =
    p_i(x_i) / q_i(x_i) from the scipy softmax: u = a -/+ 5e-7 ties, -/+ 2e-6
    does not; accept iff u < a; a draft after the first rejection is never
    tested and cannot tie."""
    for seed in range(8, 200):   # first seed whose draft 0 has a0 < 1 (a rejectable draft)
        b = make_batch(1, 2, V=64, d=16, seed=seed)
        n = _np(b)
        P, _ = _exact_p(n)
        x = n["draft_tokens"]
        q = n["draft_probs"].astype(np.float64)
        a = [P[i, x[i]] / q[i, x[i]] for i in range(2)]
        a0 = a[0]
        if 4e-6 < a0 < 0.6:
            break
    assert 4e-6 < a0 < 0.6, a
    for delta, tie in [(-2e-6, False), (-5e-7, True), (5e-7, True), (2e-6, False)]:
        u = np.array([a0 + delta, 0.0, 0.5])
        r = _verify({**n, "uniforms": u})
        assert bool(r["flags"][0] & oracle.F_ACCEPT_TIE) == tie, delta
        assert (r["accept_len"][0] >= 1) == (delta < 0)
        assert abs(r["ratio"][0] - a0) < 1e-12 * max(1.0, a0)
        margin = min(abs(delta), a[1]) if delta < 0 else abs(delta)   # test 1 (u_1 = 0) only after an accept
        assert abs(r["accept_margin"][0] - margin) < 1e-12
    # draft 1 is not tested when draft 0 is rejected: a tie at u_1 = a_1 is ignored
    u = np.array([min(a0 + 0.3, 0.999), a[1] + 1e-7, 0.5])
    r = _verify({**n, "uniforms": u})
    assert r["accept_len"][0] == 0 and not r["flags"][0] & oracle.F_ACCEPT_TIE


def test_p_tie_closed_form_uniform_p():
    """p uniform over V tokens (h = 0: every logit 0): the flagged measure of
    the final uniform is V * min(1/V, 2 eps) exactly."""
    V, d = 8, 16
    H = np.zeros((1, d), np.uint16)
    W = make_batch(1, 0, V=V, d=d, seed=1).to_numpy()["W_bits"]
    for eps, expect in [(1e-6, 8 * 2e-6), (1e-3, 8 * 2e-3), (0.1, 1.0)]:
        r = oracle.verify(H, W, np.zeros(0, np.int32), np.zeros((0, V), np.float32), np.array([0], np.int32),
                          np.array([0.3]), tie_eps=eps)
        assert abs(r["p_tie"][0] - expect) < 1e-12


@pytest.mark.parametrize("gamma", [0, 1])
def test_p_tie_monte_carlo(gamma):
    """p_tie (the probability over the uniforms that a request is flagged) is
    checked against the observed tie frequency of 20000 independent uniform
    draws of the same request (band widened to 1e-3 so ties are common);
    |freq - mean p_tie| <= 4 sigma."""
    V, d, R = 48, 16, 20000
    b = make_batch(1, gamma, V=V, d=d, seed=17)
    n = _np(b)
    H = np.tile(n["hidden_bits"], (R, 1))
    rng = np.random.default_rng(5)
    u = rng.random(R * (gamma + 1))
    x = np.tile(n["draft_tokens"], R)
    q = np.tile(n["draft_probs"], (R, 1)) if gamma else n["draft_probs"]
    r = oracle.verify(H, n["W_bits"], x, q, np.full(R, gamma, np.int32), u, tie_eps=1e-3)
    freq = r["tie"].mean()
    mean = r["p_tie"].mean()
    sd = np.sqrt(mean * (1 - mean) / R)
    assert 0.02 < mean < 0.5
    assert abs(freq - mean) <= 4 * sd + 1e-3 * gamma, (freq, mean, sd)


def test_logits_blas_matches_c_loops():
    """oracle.logits_blas (library fp64 matmul, used for full-size batches) is
    the same step-1 definition as the C loops: equal to 1e-12 relative."""
    b = make_batch(5, 1, V=3000, d=256, seed=2)
    n = _np(b)
    a = oracle.logits(n["hidden_bits"], n["W_bits"])
    c = oracle.logits_blas(n["hidden_bits"], n["W_bits"], v_chunk=777)
    assert np.max(np.abs(a - c)) <= 1e-12 * np.max(np.abs(a))
    d = oracle.logits_blas(n["hidden_bits"], n["W_bits"], W64=oracle.weight_f64(n["W_bits"]))
    assert np.max(np.abs(a - d)) <= 1e-12 * np.max(np.abs(a))


# ------------------------------------------------------------------ temperature
@pytest.mark.parametrize("T", [0.25, 2.0, 4.0])
def test_temperature_power_of_two_equals_scaled_weights(T):
    """Target at temperature T = 2^k is the T = 1 verification of W * 2^-k
    (exact in bf16 and in the fp64 logits): identical decisions and lse, so
    the temperature path is pinned to the (pinned) T = 1 path by an
    independent route."""
    import torch
    b = make_batch(20, "mixed:5", V=500, d=32, seed=31)
    n = _np(b)
    Ws = (b.W.float() / T).to(torch.bfloat16)
    assert torch.equal(Ws.float(), b.W.float() / T)
    r_t = oracle.verify(n["hidden_bits"], n["W_bits"], n["draft_tokens"], n["draft_probs"], n["gamma"],
                        n["uniforms"], temperature=T)
    r_s = oracle.verify(n["hidden_bits"], oracle.bf16_bits(Ws), n["draft_tokens"], n["draft_probs"], n["gamma"],
                        n["uniforms"])
    assert (r_t["accept_len"] == r_s["accept_len"]).all() and (r_t["next_token"] == r_s["next_token"]).all()
    assert np.array_equal(r_t["lse"], r_s["lse"])


def test_high_temperature_draws_uniformly():
    """T -> infinity: p -> uniform over V, so a gamma = 0 draw is token
    floor(u * V) (the uniform inverse CDF) away from the interval ends."""
    V = 50
    b = make_batch(200, 0, V=V, d=16, seed=4)
    n = _np(b)
    r = oracle.verify(n["hidden_bits"], n["W_bits"], np.zeros(0, np.int32), np.zeros((0, V), np.float32),
                      n["gamma"], n["uniforms"], temperature=1e9)
    u = n["uniforms"].astype(np.float64)
    far = np.abs(u * V - np.rint(u * V)) > 1e-4
    assert far.sum() > 150
    assert (r["next_token"][far] == np.floor(u[far] * V)).all()
