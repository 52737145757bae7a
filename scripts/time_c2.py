import os, sys, torch, json
sys.path.insert(0, ".")
from paper_2512_22420_b200 import NJ_OPT_PATH, NJ_PATH_FUSED, NJ_OPT_CERTIFY, Verifier
from synth.inputs import make_batch, make_weight
dev = torch.device("cuda:0")
V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
res = {}
for (B, g) in [(8, 3), (16, 2), (4, 3), (1, 0)]:
    b = make_batch(B, g, V=V, d=d, seed=0, device=dev, W=W)
    v = Verifier(d, V, max_batch=B, gamma_max=5)
    v.set_option(NJ_OPT_PATH, NJ_PATH_FUSED); v.set_option(NJ_OPT_CERTIFY, 0)
    acc = torch.empty(B, dtype=torch.int32, device=dev); nxt = torch.empty(B, dtype=torch.int32, device=dev)
    for _ in range(5): v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(30): v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
    e1.record(); torch.cuda.synchronize()
    res[f"B{B}g{g}"] = round(e0.elapsed_time(e1) / 30 * 1e3, 1)
print(os.environ.get("TAG", ""), json.dumps(res), flush=True)
