"""Raw decision accuracy of the CUDA path with the certificate OFF, at the
bench shapes: >= 10^4 Qwen-shape requests (B = 256, gamma = 5; B = 64,
gamma = 3; B = 24, gamma = 3 and B = 8, gamma = 3 on the AUTO path -- the staged
k_lmhead step with the flat one-launch sampler -- and B = 8, gamma = 3 on the
fused kernel) against
the fp64 oracle.  Counts
out-of-band mismatches (must be 0), ties (oracle band 1e-6) and excused
requests that took the other tie branch.  Writes one JSON summary.

    python scripts/uncertified_sweep.py [--batches 40] [--out profiles/r02_uncertified.json]
"""
import argparse
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle  # noqa: E402
import parity  # noqa: E402
from paper_2512_22420_b200 import NJ_OPT_CERTIFY, NJ_OPT_PATH, NJ_PATH_AUTO, NJ_PATH_FUSED, Verifier  # noqa: E402
from synth.inputs import make_batch, make_weight  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batches", type=int, default=40)
ap.add_argument("--out", default="profiles/r02c_uncertified.json")
a = ap.parse_args()
dev = torch.device("cuda:0")
V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
W64 = oracle.weight_f64(oracle.bf16_bits(W))
summary = {}
t0 = time.time()
for (B, g, nb, fp) in [(256, 5, a.batches, NJ_PATH_AUTO), (64, 3, a.batches, NJ_PATH_AUTO),
                      (24, 3, 2 * a.batches, NJ_PATH_AUTO),   # the flat one-launch sampler's range
                      (8, 3, 4 * a.batches, NJ_PATH_AUTO), (8, 3, 2 * a.batches, NJ_PATH_FUSED)]:
    v = Verifier(d, V, max_batch=B, gamma_max=5)
    v.set_option(NJ_OPT_CERTIFY, 0)
    v.set_option(NJ_OPT_PATH, fp)
    path = v.plan(np.full(B, g, np.int32))[0]
    tot = {"requests": 0, "mismatch_out_of_band": 0, "ties": 0, "expected_ties": 0.0, "excused_other_branch": 0}
    for i in range(nb):
        b = make_batch(B, g, V=V, d=d, seed=5000 + 97 * B + i, device=dev, W=W)
        acc = torch.empty(B, dtype=torch.int32, device=dev)
        nxt = torch.empty(B, dtype=torch.int32, device=dev)
        v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
        torch.cuda.synchronize()
        n = b.to_numpy()
        L = oracle.logits_blas(n["hidden_bits"], None, W64=W64)
        r = oracle.verify_from_logits(L, n["draft_tokens"], n["draft_probs"], n["gamma"], n["uniforms"])
        a_, t_ = acc.cpu().numpy(), nxt.cpu().numpy()
        bad = ~r["tie"] & ((a_ != r["accept_len"]) | (t_ != r["next_token"]))
        tot["requests"] += B
        tot["mismatch_out_of_band"] += int(bad.sum())
        tot["ties"] += int(r["tie"].sum())
        tot["expected_ties"] += float(r["p_tie"].sum())
        try:
            parity.check(f"sweep B={B} g={g} p={fp} #{i}", n, a_, t_, r=r, L=L)
        except AssertionError as e:
            tot.setdefault("failures", []).append(str(e)[:300])
        tot["excused_other_branch"] = sum(s["excused_differing"] for s in parity.STATS
                                          if s["test"].startswith(f"sweep B={B} g={g} p={fp}"))
    tot["path"] = ["auto", "fused", "two-pass", "staged"][path]
    key = f"B{B}_g{g}" + ("_fused" if fp == NJ_PATH_FUSED else "")
    summary[key] = tot
    print(json.dumps({key: tot}), flush=True)
summary["total_requests"] = sum(v_["requests"] for v_ in summary.values() if isinstance(v_, dict))
summary["total_mismatch_out_of_band"] = sum(v_["mismatch_out_of_band"] for v_ in summary.values() if isinstance(v_, dict))
summary["certificate"] = "off (raw kernels)"
summary["seconds"] = time.time() - t0
json.dump(summary, open(a.out, "w"), indent=1)
print(json.dumps({k: summary[k] for k in ("total_requests", "total_mismatch_out_of_band", "seconds")}))
