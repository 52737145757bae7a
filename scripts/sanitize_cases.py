"""Small verification calls for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): every nj_verify path (fused, staged, two-pass), the
certified fp64 fallback (forced), a 4-shard vocab-sharded group, the proposal
step and greedy verification, each once on small shapes, plus (--c2) one call
at the C2 shape.  Decisions are checked against the oracle so a sanitizer run
that perturbs timing still verifies results.

    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py [--c2]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2512_22420_b200 import (NJ_OPT_FORCE_FALLBACK, NJ_OPT_PATH, NJ_PATH_FUSED, NJ_PATH_STAGED,  # noqa: E402
                                   NJ_PATH_TWOPASS, ShardGroup, Verifier)
from synth.inputs import make_batch, make_weight  # noqa: E402

dev = torch.device("cuda:0")


def check(b, acc, nxt):
    n = b.to_numpy()
    r = oracle.verify(n["hidden_bits"], n["W_bits"], n["draft_tokens"], n["draft_probs"], n["gamma"], n["uniforms"])
    ok = ~r["tie"]
    a, t = acc.cpu().numpy(), nxt.cpu().numpy()
    assert (a[ok] == r["accept_len"][ok]).all() and (t[ok] == r["next_token"][ok]).all()


def run(b, path, force_fb=False):
    v = Verifier(b.hidden.shape[1], b.W.shape[0], max_batch=b.B, gamma_max=5)
    v.set_option(NJ_OPT_PATH, path)
    v.set_option(NJ_OPT_FORCE_FALLBACK, int(force_fb))
    acc = torch.full((b.B,), -7, dtype=torch.int32, device=dev)
    nxt = torch.full((b.B,), -7, dtype=torch.int32, device=dev)
    v.verify(b.hidden, b.W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
    torch.cuda.synchronize()
    check(b, acc, nxt)
    v.close()


cases = []
for name, B, g, V, d, path, fb in [("fused", 6, "mixed:5", 2048, 128, NJ_PATH_FUSED, False),
                                   ("staged", 16, 3, 2048, 128, NJ_PATH_STAGED, False),
                                   ("twopass", 10, "mixed:5", 2048, 128, NJ_PATH_TWOPASS, False),
                                   ("fallback", 4, "mixed:3", 1024, 64, NJ_PATH_TWOPASS, True)]:
    b = make_batch(B, g, V=V, d=d, seed=B, device=dev)
    run(b, path, fb)
    print(name, "ok", flush=True)
# k_lmhead in both CTA-group modes, several token chunks, ragged vocab / rows (staged path)
import os  # noqa: E402
for cg in ("1", "2"):
    os.environ["NJ_LM_CG"] = cg
    b = make_batch(75, 3, V=4093, d=256, seed=11, device=dev)   # N = 300: 3 (CTA) / 2 (pair) chunks
    run(b, NJ_PATH_STAGED)
    print("staged k_lmhead cg" + cg, "ok", flush=True)
os.environ.pop("NJ_LM_CG", None)
# k_sample_small (staged, B <= 12: one cluster of 8 CTAs per request, DSMEM chunk masses),
# 10 chunks of 4096 ids (several per CTA, ragged last chunk)
b = make_batch(7, "mixed:5", V=40000, d=64, seed=13, device=dev)
run(b, NJ_PATH_STAGED)
print("staged small-batch sampler ok", flush=True)
# forced cluster sizes: 12 / 2 CTAs per request, 25 chunks (2 CTAs: 5 staged batches, the owner
# re-reads its chunk from global memory; 12: one batch, read from the staging buffer)
for cl in ("12", "2"):
    os.environ["NJ_SMALL_CL"] = cl
    b = make_batch(5, "mixed:4", V=100000, d=64, seed=14, device=dev)
    run(b, NJ_PATH_STAGED)
    print("staged small-batch sampler cl" + cl, "ok", flush=True)
os.environ.pop("NJ_SMALL_CL", None)
b = make_batch(6, "mixed:4", V=2048, d=128, seed=5, device=dev)
grp = ShardGroup(128, 2048, max_batch=6, gamma_max=5, nshards=4)
acc = torch.empty(6, dtype=torch.int32, device=dev)
nxt = torch.empty(6, dtype=torch.int32, device=dev)
grp.verify(b.hidden, grp.shards(b.W), b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
torch.cuda.synchronize()
check(b, acc, nxt)
grp.close()
print("sharded4 ok", flush=True)
b = make_batch(5, 0, V=2048, d=128, seed=11, device=dev)
v = Verifier(128, 2048, max_batch=6, gamma_max=5)
tok = torch.empty(5, dtype=torch.int32, device=dev)
q = torch.empty(5, 2048, device=dev)
v.propose(b.hidden, b.W, b.uniforms, tok, q)
b2 = make_batch(6, "mixed:5", V=2048, d=128, seed=12, device=dev)
acc = torch.empty(6, dtype=torch.int32, device=dev)
nxt = torch.empty(6, dtype=torch.int32, device=dev)
v.verify_greedy(b2.hidden, b2.W, b2.draft_tokens, b2.gamma, acc, nxt)
torch.cuda.synchronize()
print("propose/greedy ok", flush=True)
if "--c2" in sys.argv:
    W = make_weight(152064, 3584, 0, dev)
    b = make_batch(8, 3, V=152064, d=3584, seed=100, device=dev, W=W)
    run(b, NJ_PATH_FUSED)
    print("c2 fused ok", flush=True)
    run(b, NJ_PATH_STAGED)   # k_lmhead (one CTA chunk, 2-k-block stages) + k_sample_small
    print("c2 staged ok", flush=True)
print("all cases ok")
