"""Write tests/golden/c1_fixed_uniforms.json: BJ config 1 (B=1, gamma=3,
V=32, d=16) evaluated by the fp64 oracle ONLY, at uniforms that force each
acceptance length (SURVEY §8(c) "forced branches": u=0 accepts a draft with
p > 0, u=1-2^-24 rejects it unless a = p/q > 1-2^-24) plus random draws.

The seed is the first one from 1234 up whose three drafts all have a_i < 1 so
that the forced rejections really reject; the script asserts that the cases
hit every acceptance length n = 0, 1, 2, 3 (residual draws from
max(0, p_n - q_n) for n < 3, the bonus draw for n = 3)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from synth.inputs import make_batch  # noqa: E402

top = float(np.float32(1.0 - 2.0 ** -24))
SEED = 1234
while True:
    b = make_batch(1, 3, V=32, d=16, seed=SEED)
    n = b.to_numpy()
    r0 = oracle.verify(n["hidden_bits"], n["W_bits"], n["draft_tokens"], n["draft_probs"], n["gamma"],
                       np.array([0.0, 0.0, 0.0, 0.5], np.float32))
    if (r0["ratio"] < top).all():
        break
    SEED += 1
cases = []
rng = np.random.default_rng(SEED)
for k in range(4):
    for draw in [0.0, 0.25, 0.5, 0.75, top]:
        u = np.array([0.0] * k + [top] * (3 - k) + [draw], np.float32)
        r = oracle.verify(n["hidden_bits"], n["W_bits"], n["draft_tokens"], n["draft_probs"], n["gamma"], u)
        if r["tie"][0]:
            continue
        cases.append({"uniforms": [float(x) for x in u], "accept_len": int(r["accept_len"][0]),
                      "next_token": int(r["next_token"][0])})
for _ in range(12):
    u = (rng.integers(0, 1 << 24, size=4) * 2.0 ** -24).astype(np.float32)
    r = oracle.verify(n["hidden_bits"], n["W_bits"], n["draft_tokens"], n["draft_probs"], n["gamma"], u)
    if r["tie"][0]:
        continue
    cases.append({"uniforms": [float(x) for x in u], "accept_len": int(r["accept_len"][0]),
                  "next_token": int(r["next_token"][0])})
assert sorted({c["accept_len"] for c in cases}) == [0, 1, 2, 3], cases
out = {"source": "scripts/make_golden.py (oracle/ only); BASELINE.json configs[0]", "seed": SEED,
       "V": 32, "d": 16, "gamma": 3, "cases": cases}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                    "c1_fixed_uniforms.json")
json.dump(out, open(path, "w"), indent=1)
print(path, len(cases))
