import json, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import oracle
from paper_2512_22420_b200 import NJ_OPT_PATH, NJ_PATH_FUSED, NJ_OPT_CERTIFY, Verifier
from synth.inputs import make_batch, make_weight
dev = torch.device("cuda:0")
V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
v = Verifier(d, V, max_batch=48, gamma_max=5)
v.set_option(NJ_OPT_PATH, NJ_PATH_FUSED)
tot = {"req": 0, "mis_acc": 0, "mis_tok": 0, "ties": 0, "fallback": 0, "lse_err": 0.0, "lnp_err": 0.0, "mass_rel": 0.0}
cases = [(8, 3, s) for s in range(6)] + [(8, "mixed:5", 100 + s) for s in range(3)] + [(1, 0, 7), (48, 0, 8), (16, 2, 9), (12, 3, 10)]
t0 = time.time()
for B, g, seed in cases:
    b = make_batch(B, g, V=V, d=d, seed=seed, device=dev, W=W)
    if b.N > 48: continue
    acc = torch.empty(B, dtype=torch.int32, device=dev); nxt = torch.empty(B, dtype=torch.int32, device=dev)
    dd = {"lse": torch.full((b.N,), float("nan"), device=dev), "p_draft": torch.zeros(max(b.G, 1), device=dev),
          "mass": torch.zeros(B, dtype=torch.float64, device=dev), "flags": torch.zeros(B, dtype=torch.int32, device=dev)}
    v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt, debug=dd)
    torch.cuda.synchronize()
    n = b.to_numpy()
    r = oracle.verify(n["hidden_bits"], n["W_bits"], n["draft_tokens"], n["draft_probs"], n["gamma"], n["uniforms"])
    a, t = acc.cpu().numpy(), nxt.cpu().numpy()
    ok = ~r["tie"]
    fl = dd["flags"].cpu().numpy()
    tot["req"] += B; tot["ties"] += int(r["tie"].sum()); tot["fallback"] += int((fl & 1).sum())
    tot["mis_acc"] += int(((a != r["accept_len"]) & ok).sum()); tot["mis_tok"] += int(((t != r["next_token"]) & ok).sum())
    tot["lse_err"] = max(tot["lse_err"], float(np.abs(dd["lse"].cpu().numpy() - r["lse"]).max()))
    if b.G:
        m = r["p_draft"] > 1e-30
        pg = dd["p_draft"].cpu().numpy()[:b.G]
        tot["lnp_err"] = max(tot["lnp_err"], float(np.abs(np.log(np.maximum(pg[m], 1e-38)) - np.log(r["p_draft"][m])).max()))
    tot["mass_rel"] = max(tot["mass_rel"], float(np.max(np.abs(dd["mass"].cpu().numpy() - r["mass"]) / r["mass"])))
    print(B, g, seed, "mis", int(((a != r["accept_len"]) & ok).sum()), int(((t != r["next_token"]) & ok).sum()), "fl", fl.tolist(), flush=True)
tot["secs"] = time.time() - t0
# timing at C2 (certify on = production)
b = make_batch(8, 3, V=V, d=d, seed=0, device=dev, W=W)
acc = torch.empty(8, dtype=torch.int32, device=dev); nxt = torch.empty(8, dtype=torch.int32, device=dev)
for c in (1, 0):
    v.set_option(NJ_OPT_CERTIFY, c)
    for _ in range(5): v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(30): v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
    e1.record(); torch.cuda.synchronize()
    tot[f"c2_us_certify{c}"] = e0.elapsed_time(e1) / 30 * 1e3
print(json.dumps(tot))
json.dump(tot, open("gpurun_out/fused_sweep.json", "w"))
