import os, sys, torch, json, numpy as np
sys.path.insert(0, ".")
from paper_2512_22420_b200 import NJ_OPT_PATH, NJ_PATH_TWOPASS, NJ_OPT_CERTIFY, NJ_OPT_PROFILE, Verifier
from synth.inputs import make_batch, make_weight
dev = torch.device("cuda:0"); V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
res = {}
for (B, g) in [(16, 3), (32, 3), (64, 3), (256, 2), (256, 5)]:
    b = make_batch(B, g, V=V, d=d, seed=1, device=dev, W=W)
    v = Verifier(d, V, max_batch=B, gamma_max=5); v.set_option(NJ_OPT_PATH, NJ_PATH_TWOPASS)
    acc = torch.empty(B, dtype=torch.int32, device=dev); nxt = torch.empty(B, dtype=torch.int32, device=dev)
    fl = torch.zeros(B, dtype=torch.int32, device=dev)
    out = {}
    for c in (1, 0):
        v.set_option(NJ_OPT_CERTIFY, c)
        for _ in range(3): v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt, debug={"flags": fl})
        torch.cuda.synchronize()
        if c: out["fallback_frac"] = float((fl.cpu().numpy() & 1).mean())
        v.set_option(NJ_OPT_PROFILE, 1); v.kernel_time(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
        e1.record(); torch.cuda.synchronize()
        out[f"us_certify{c}"] = round(e0.elapsed_time(e1) / 5 * 1e3, 1)
        kms, kn = v.kernel_time(True); v.set_option(NJ_OPT_PROFILE, 0)
        out[f"KA_us_certify{c}"] = round(kms / max(kn, 1) * 1e3, 1)
    res[f"B{B}g{g}"] = out
    print(B, g, out, flush=True)
    del v
