"""CPU checks of tests/parity.py, the band-aware comparison the GPU parity
tests use for excused (near-tie) requests (R12): the alternative
outcomes it accepts are exactly the other branches of the tied decisions."""
import numpy as np

import oracle
import parity
from synth.inputs import make_batch


def _logits(n):
    return oracle.logits(n["hidden_bits"], n["W_bits"])


def test_valid_outcomes_draw_tie_adds_neighbour():
    b = make_batch(1, 0, V=64, d=16, seed=21)
    n = b.to_numpy()
    L = _logits(n)
    r = oracle.verify_from_logits(L, np.zeros(0, np.int32), np.zeros((0, 64), np.float32), [0], [0.3])
    hi = r["F_hi"][0]
    t = r["next_token"][0]
    u = np.array([hi - 4e-7])
    outs = parity.valid_outcomes(L, np.zeros(0, np.int32), np.zeros((1, 64), np.float32), 0, u)
    assert outs == {(0, t), (0, t + 1)}
    outs = parity.valid_outcomes(L, np.zeros(0, np.int32), np.zeros((1, 64), np.float32), 0, np.array([hi - 3e-6]))
    assert outs == {(0, t)}


def test_valid_outcomes_accept_tie_adds_other_branch():
    for seed in range(8, 200):
        b = make_batch(1, 2, V=64, d=16, seed=seed)
        n = b.to_numpy()
        L = _logits(n)
        r = oracle.verify_from_logits(L, n["draft_tokens"], n["draft_probs"], [2], [0.0, 0.0, 0.5])
        if 1e-3 < r["ratio"][0] < 0.6:
            break
    a0 = r["ratio"][0]
    u = np.array([a0 + 3e-7, 0.0, 0.5])          # rejects at 0, within the band
    outs = parity.valid_outcomes(L, n["draft_tokens"], n["draft_probs"], 2, u)
    rej = oracle.verify_from_logits(L, n["draft_tokens"], n["draft_probs"], [2], np.array([1.5, 0.0, 0.5]))
    acc = oracle.verify_from_logits(L, n["draft_tokens"], n["draft_probs"], [2], np.array([0.0, 0.0, 0.5]))
    assert (int(rej["accept_len"][0]), int(rej["next_token"][0])) in outs
    assert (int(acc["accept_len"][0]), int(acc["next_token"][0])) in outs
    assert int(acc["accept_len"][0]) >= 1 and int(rej["accept_len"][0]) == 0


def test_check_flags_out_of_band_mismatch():
    b = make_batch(6, "mixed:3", V=200, d=16, seed=3)
    n = b.to_numpy()
    r = oracle.verify(n["hidden_bits"], n["W_bits"], n["draft_tokens"], n["draft_probs"], n["gamma"], n["uniforms"])
    parity.check("helper/self", n, r["accept_len"], r["next_token"])
    bad = r["next_token"].copy()
    k = int(np.nonzero(~r["tie"])[0][0])
    bad[k] = (bad[k] + 1) % 200
    try:
        parity.check("helper/bad", n, r["accept_len"], bad)
    except AssertionError:
        return
    raise AssertionError("a wrong token outside the band was not caught")
