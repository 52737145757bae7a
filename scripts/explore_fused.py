"""Fused-path step time under knobs: NJ_SACC (one partial per ring stage),
NJ_KPD (k-blocks per partial, single-buffer mode), NJ_KGROUP.  Certificate on
(as in bench) and uncertified decision parity vs the oracle at C2."""
import os, sys, json, torch, numpy as np
sys.path.insert(0, ".")
from paper_2512_22420_b200 import NJ_OPT_CERTIFY, NJ_OPT_PATH, NJ_OPT_PROFILE, Verifier
from synth.inputs import make_batch, make_weight
import oracle
dev = torch.device("cuda:0"); V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
KN = ["NJ_SACC", "NJ_KPD", "NJ_KGROUP", "NJ_FGROUPS", "NJ_GRID"]
for (B, g) in [(8, 3), (1, 0)]:
    b = make_batch(B, g, V=V, d=d, seed=11, device=dev, W=W)
    ref = None
    for var in [{}, {"NJ_GRID": "148"}, {"NJ_GRID": "144"}, {"NJ_GRID": "140"}]:
        for k in KN: os.environ.pop(k, None)
        os.environ.update(var)
        v = Verifier(d, V, max_batch=B, gamma_max=5); v.set_option(NJ_OPT_PATH, 1)
        acc = torch.empty(B, dtype=torch.int32, device=dev); nxt = torch.empty(B, dtype=torch.int32, device=dev)
        pd = torch.zeros(max(b.G, 1), device=dev)
        v.set_option(NJ_OPT_CERTIFY, 0)
        v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt, debug={"p_draft": pd})
        torch.cuda.synchronize()
        if ref is None and b.G:
            n = b.to_numpy()
            ref = oracle.verify(n["hidden_bits"], n["W_bits"], n["draft_tokens"], n["draft_probs"], n["gamma"], n["uniforms"])
        lnp = float(np.abs(np.log(pd.cpu().numpy()[:b.G]) - np.log(ref["p_draft"])).max()) if b.G else 0.0
        v.set_option(NJ_OPT_CERTIFY, 1)
        for _ in range(3): v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
        e1.record(); torch.cuda.synchronize()
        print(f"B{B}g{g} N={b.N} {var} us={e0.elapsed_time(e1) / 20 * 1e3:.1f} max|dlnp|={lnp:.2e}", flush=True)
        del v
