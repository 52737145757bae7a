"""Dominant-kernel time vs accumulator-restart period (NJ_KS) for the staged
(N=256) and two-pass (B=256, gamma=5) paths."""
import os, sys, json, torch
sys.path.insert(0, ".")
from paper_2512_22420_b200 import NJ_OPT_CERTIFY, NJ_OPT_PROFILE, Verifier
from synth.inputs import make_batch, make_weight
dev = torch.device("cuda:0"); V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
out = {}
for (B, g) in [(64, 3), (256, 5)]:
    b = make_batch(B, g, V=V, d=d, seed=5, device=dev, W=W)
    for ks in [int(x) for x in sys.argv[1].split(",")]:
        os.environ["NJ_KS"] = str(ks)
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
        out[f"B{B}g{g}_ks{ks}"] = (round(e0.elapsed_time(e1) / 10 * 1e3, 1), round(kms / kn * 1e3, 1))
        print(f"B{B}g{g}_ks{ks}", out[f"B{B}g{g}_ks{ks}"], flush=True)
        del v
