"""Staged-path GEMM (all N rows, logits staged in L2) time under the token-chunk
knob (NJ_BIG_MAXT; chunks <= 128 columns use two epilogue teams) at N = 192-512."""
import os, sys, json, torch
sys.path.insert(0, ".")
from paper_2512_22420_b200 import NJ_OPT_CERTIFY, NJ_OPT_PROFILE, NJ_OPT_PATH, NJ_PATH_STAGED, Verifier
from synth.inputs import make_batch, make_weight
dev = torch.device("cuda:0"); V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
out = {}
for (B, g) in [(48, 3), (64, 3), (96, 3), (128, 3)]:
    b = make_batch(B, g, V=V, d=d, seed=5, device=dev, W=W)
    for var in [{}, {"NJ_BIG_MAXT": "128"}, {"NJ_BIG_MAXT": "96"}, {"NJ_BIG_MAXT": "64"}, {}]:
        os.environ.pop("NJ_BIG_MAXT", None)
        os.environ.update(var)
        try:
            v = Verifier(d, V, max_batch=B, gamma_max=5); v.set_option(NJ_OPT_CERTIFY, 0)
            v.set_option(NJ_OPT_PATH, NJ_PATH_STAGED)
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
        key = f"B{B}g{g} " + (",".join(f"{k}={v_}" for k, v_ in var.items()) or "default")
        out[key] = r
        print(key, r, flush=True)
json.dump(out, open("gpurun_out/explore_staged.json", "w"), indent=1)
