"""k_gemm_big: logit accuracy vs fp64 at several accumulator-restart periods
(NJ_KS k-blocks) and step timings vs the old k_gemm_acc (NJ_GEMM=acc).
Writes gpurun_out/big_check.json."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2512_22420_b200 import NJ_OPT_CERTIFY, NJ_OPT_PATH, NJ_OPT_PROFILE, NJ_PATH_STAGED, NJ_PATH_TWOPASS, Verifier
from synth.inputs import make_batch, make_weight
dev = torch.device("cuda:0")
V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
res = {"acc": {}, "time": {}}


def run(v, b, dbg=None, n=1):
    acc = torch.empty(b.B, dtype=torch.int32, device=dev); nxt = torch.empty(b.B, dtype=torch.int32, device=dev)
    for _ in range(n):
        v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt, debug=dbg)
    return acc, nxt


# accuracy: staged path (all rows' lse) at N = 256, two-pass at N = 512
for name, (B, g, path) in {"staged_b64g3": (64, 3, NJ_PATH_STAGED), "twopass_b128g3": (128, 3, NJ_PATH_TWOPASS)}.items():
    b = make_batch(B, g, V=V, d=d, seed=3, device=dev, W=W)
    ref_l = (b.hidden.double() @ W.double().t())
    lse_ref = torch.logsumexp(ref_l, 1)
    gi = torch.from_numpy(np.concatenate([np.arange(ro, ro + gg) for ro, gg in
                                          zip(np.concatenate([[0], np.cumsum(b.gamma + 1)[:-1]]), b.gamma)])).to(dev).long()
    tok = b.draft_tokens.long()
    lnp_ref = ref_l[gi, tok] - lse_ref[gi]
    del ref_l
    for ks in (1, 2, 4, 8, 16):
        os.environ["NJ_KS"] = str(ks)
        v = Verifier(d, V, max_batch=B, gamma_max=5)
        v.set_option(NJ_OPT_PATH, path); v.set_option(NJ_OPT_CERTIFY, 0)
        dbg = {"lse": torch.full((b.N,), float("nan"), device=dev), "p_draft": torch.zeros(b.G, device=dev)}
        run(v, b, dbg)
        torch.cuda.synchronize()
        fin = torch.isfinite(dbg["lse"])
        lse_err = (dbg["lse"].double() - lse_ref)[fin].abs()
        lnp = torch.log(dbg["p_draft"].double().clamp_min(1e-38))
        m = lnp_ref > -20
        lnp_err = (lnp - lnp_ref)[m].abs()
        p_ref = lnp_ref.exp()
        res["acc"][f"{name}_ks{ks}"] = {"lse_err_max": float(lse_err.max()), "lse_err_mean": float(lse_err.mean()),
                                        "lse_bias": float((dbg["lse"].double() - lse_ref)[fin].mean()),
                                        "lnp_err_max": float(lnp_err.max()),
                                        "lnp_err_max_p_gt_1e-3": float((lnp - lnp_ref)[p_ref > 1e-3].abs().max()),
                                        "rows": int(fin.sum())}
        print(name, ks, res["acc"][f"{name}_ks{ks}"], flush=True)
        del v
os.environ["NJ_KS"] = "4"

# timings (certificate on, default path choice), new vs old GEMM
pts = [(16, 3), (32, 3), (64, 3), (128, 1), (64, 5), (128, 3), (256, 1), (256, 2), (128, 5), (256, 3), (256, 5), (256, "mixed:5")]
for kind in ("big", "acc"):
    if kind == "acc":
        os.environ["NJ_GEMM"] = "acc"
    for B, g in pts:
        b = make_batch(B, g, V=V, d=d, seed=5, device=dev, W=W)
        v = Verifier(d, V, max_batch=B, gamma_max=5)
        path, _ = v.plan(b.gamma)
        fl = torch.zeros(B, dtype=torch.int32, device=dev)
        run(v, b, {"flags": fl}, 3)
        torch.cuda.synchronize()
        fb = float((fl.cpu().numpy() & 1).mean())
        v.set_option(NJ_OPT_PROFILE, 1); v.kernel_time(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); run(v, b, None, 10); e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 10 * 1e3
        kms, kn = v.kernel_time(True)
        key = f"{kind}_B{B}_g{g}"
        res["time"][key] = {"N": b.N, "path": int(path), "us": us, "dom_us": kms / max(kn, 1) * 1e3, "fallback_frac": fb,
                            "pos_per_s": b.N / us * 1e6}
        print(key, res["time"][key], flush=True)
        del v
json.dump(res, open("gpurun_out/big_check.json", "w"), indent=1)
