"""Dominant-kernel time of k_gemm_big under tuning knobs (env): stages, k-blocks
per stage, token chunk, L2 prefetch distance, CTA pair.  Certificate off."""
import os, sys, json, itertools, torch
sys.path.insert(0, ".")
from paper_2512_22420_b200 import NJ_OPT_CERTIFY, NJ_OPT_PROFILE, Verifier
from synth.inputs import make_batch, make_weight
dev = torch.device("cuda:0"); V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
KNOBS = ["NJ_CG", "NJ_PF", "NJ_BIG_S", "NJ_BIG_GK", "NJ_BIG_MAXT", "NJ_KS", "NJ_BIG_DBG", "NJ_SPIN", "NJ_SLEEP", "NJ_BIG_NBUF", "NJ_TEAMS", "NJ_KS_KA", "NJ_W_EVICT_FIRST", "NJ_STATS"]
variants = [{}, {"NJ_STATS": "0"}, {}, {"NJ_STATS": "0"}]
out = {}
for (B, g) in [(16, 3), (64, 3), (256, 5)]:
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
        key = f"B{B}g{g} " + ",".join(f"{k}={v_}" for k, v_ in var.items())
        out[key] = r
        print(key, r, flush=True)
json.dump(out, open("gpurun_out/explore_big.json", "w"), indent=1)
