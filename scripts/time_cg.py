"""Step / dominant-kernel time of k_gemm_big with single CTAs (NJ_CG=1) vs CTA
pairs (NJ_CG=2) across the staged / two-pass regime, plus a parity spot check
(uncertified decisions vs the unsharded CG=1 run)."""
import os, sys, json, torch
sys.path.insert(0, ".")
from paper_2512_22420_b200 import NJ_OPT_CERTIFY, NJ_OPT_PROFILE, Verifier
from synth.inputs import make_batch, make_weight
dev = torch.device("cuda:0"); V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
out = {}
pts = [(16, 3), (32, 3), (64, 3), (48, 5), (128, 3), (256, 2), (256, 3), (256, 5)]
for (B, g) in pts:
    b = make_batch(B, g, V=V, d=d, seed=5, device=dev, W=W)
    res = {}
    for cg in (1, 2):
        os.environ["NJ_CG"] = str(cg)
        v = Verifier(d, V, max_batch=B, gamma_max=5); v.set_option(NJ_OPT_CERTIFY, 0)
        acc = torch.empty(B, dtype=torch.int32, device=dev); nxt = torch.empty(B, dtype=torch.int32, device=dev)
        lse = torch.full((b.N,), float("nan"), device=dev)
        v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt, debug={"lse": lse})
        torch.cuda.synchronize()
        res[cg] = (acc.cpu().clone(), nxt.cpu().clone(), lse.cpu().clone())
        for _ in range(2): v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
        torch.cuda.synchronize()
        v.set_option(NJ_OPT_PROFILE, 1); v.kernel_time(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
        e1.record(); torch.cuda.synchronize()
        kms, kn = v.kernel_time(True)
        out[f"B{B}g{g}_cg{cg}"] = (round(e0.elapsed_time(e1) / 10 * 1e3, 1), round(kms / kn * 1e3, 1))
        del v
    a1, n1, l1 = res[1]; a2, n2, l2 = res[2]
    fin = torch.isfinite(l1) & torch.isfinite(l2)
    out[f"B{B}g{g}_same"] = (bool((a1 == a2).all()), int((n1 != n2).sum()), float((l1 - l2)[fin].abs().max()))
    print(f"B{B}g{g}", out[f"B{B}g{g}_cg1"], out[f"B{B}g{g}_cg2"], out[f"B{B}g{g}_same"], flush=True)
json.dump(out, open("gpurun_out/time_cg.json", "w"), indent=1)
