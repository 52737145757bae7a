"""K-A (two-pass, B=256, gamma=5) time under k_gemm_big knobs (env): token
chunk width, ring stages, k-blocks per stage, accumulator buffers.  Certificate off."""
import os, sys, json, torch
sys.path.insert(0, ".")
from paper_2512_22420_b200 import NJ_OPT_CERTIFY, NJ_OPT_PROFILE, Verifier
from synth.inputs import make_batch, make_weight
dev = torch.device("cuda:0"); V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
KNOBS = ["NJ_BIG_S", "NJ_BIG_GK", "NJ_BIG_MAXT", "NJ_BIG_NBUF", "NJ_TEAMS", "NJ_KS_KA"]
variants = [{}, {"NJ_BIG_MAXT": "128"}, {"NJ_BIG_MAXT": "192"}, {"NJ_BIG_MAXT": "160"}, {"NJ_BIG_S": "3"},
            {"NJ_BIG_GK": "1"}, {"NJ_BIG_GK": "3"}, {"NJ_BIG_GK": "1", "NJ_BIG_S": "4"}, {"NJ_BIG_MAXT": "128", "NJ_TEAMS": "0"},
            {"NJ_BIG_MAXT": "192", "NJ_BIG_GK": "3"}, {"NJ_KS_KA": "16"}, {}]
out = {}
B, g = 256, 5
b = make_batch(B, g, V=V, d=d, seed=5, device=dev, W=W)
for var in variants:
    for k in KNOBS:
        os.environ.pop(k, None)
    os.environ.update(var)
    try:
        v = Verifier(d, V, max_batch=B, gamma_max=5); v.set_option(NJ_OPT_CERTIFY, 0)
        acc = torch.empty(B, dtype=torch.int32, device=dev); nxt = torch.empty(B, dtype=torch.int32, device=dev)
        for _ in range(3): v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
        torch.cuda.synchronize()
        v.set_option(NJ_OPT_PROFILE, 1); v.kernel_time(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
        e1.record(); torch.cuda.synchronize()
        kms, kn = v.kernel_time(True)
        r = (round(e0.elapsed_time(e1) / 10 * 1e3, 1), round(kms / kn * 1e3, 1))
        del v
    except Exception as e:
        r = str(e)[:100]
    key = ",".join(f"{k}={v_}" for k, v_ in var.items()) or "default"
    out[key] = r
    print(key, r, flush=True)
json.dump(out, open("gpurun_out/explore_ka.json", "w"), indent=1)
