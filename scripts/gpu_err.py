"""Error structure of the tcgen05 LM-head logits vs an fp64 reference, and
certificate-off timings of both paths."""
import json, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2512_22420_b200 import NJ_OPT_CERTIFY, NJ_OPT_PATH, NJ_PATH_FUSED, NJ_PATH_TWOPASS, Verifier
from synth.inputs import make_batch, make_weight
dev = torch.device("cuda:0")
V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
b = make_batch(8, 3, V=V, d=d, seed=11, device=dev, W=W)
R = b.N
v = Verifier(d, V, max_batch=64, gamma_max=5)
rows = torch.arange(R, dtype=torch.int32, device=dev)
L = torch.empty(R, V, device=dev)
v.lmhead_logits(b.hidden, W, rows, L)
torch.cuda.synchronize()
Ld = b.hidden.double() @ W.double().t()
dl = (L.double() - Ld)
res = {}
# per-row regression dl = a + k*l
ks, a_s, rs = [], [], []
for r in range(R):
    x = Ld[r]; y = dl[r]
    A = torch.stack([torch.ones_like(x), x], 1)
    sol = torch.linalg.lstsq(A, y[:, None]).solution[:, 0]
    ks.append(float(sol[1])); a_s.append(float(sol[0])); rs.append(float((y - A @ sol).std()))
res["kappa_mean"] = float(np.mean(ks)); res["kappa_range"] = [float(np.min(ks)), float(np.max(ks))]
res["resid_std"] = float(np.mean(rs)); res["dl_max"] = float(dl.abs().max()); res["dl_std"] = float(dl.std())
res["l_std"] = float(Ld.std())
# lse / p errors and CDF error at random u for bonus rows
lse_g = torch.logsumexp(L.double(), 1); lse_d = torch.logsumexp(Ld, 1)
res["lse_err_max"] = float((lse_g - lse_d).abs().max())
Pg = torch.softmax(L.double(), 1); Pd = torch.softmax(Ld, 1)
Fg = torch.cumsum(Pg, 1); Fd = torch.cumsum(Pd, 1)
res["F_err_max"] = float((Fg - Fd).abs().max()); res["F_err_mean"] = float((Fg - Fd).abs().mean())
# p ratio error at random tokens weighted by p
res["lnp_err_at_top"] = float((torch.log(Pg.max(1).values) - torch.log(Pd.max(1).values)).abs().max())
# timings, certificate off
tim = {}
for name, (B, g, path) in {"fused_c2": (8, 3, NJ_PATH_FUSED), "twopass_c2": (8, 3, NJ_PATH_TWOPASS),
                           "twopass_b64g3": (64, 3, NJ_PATH_TWOPASS), "twopass_b256g2": (256, 2, NJ_PATH_TWOPASS),
                           "twopass_b256g5": (256, 5, NJ_PATH_TWOPASS)}.items():
    bb = make_batch(B, g, V=V, d=d, seed=5, device=dev, W=W)
    vv = Verifier(d, V, max_batch=B, gamma_max=5)
    vv.set_option(NJ_OPT_PATH, path); vv.set_option(NJ_OPT_CERTIFY, 0)
    acc = torch.empty(B, dtype=torch.int32, device=dev); nxt = torch.empty(B, dtype=torch.int32, device=dev)
    for _ in range(3):
        vv.verify(bb.hidden, W, bb.draft_tokens, bb.draft_probs, bb.gamma, bb.uniforms, acc, nxt)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        vv.verify(bb.hidden, W, bb.draft_tokens, bb.draft_probs, bb.gamma, bb.uniforms, acc, nxt)
    e1.record(); torch.cuda.synchronize()
    tim[name] = e0.elapsed_time(e1) / 10 * 1e3
    del vv
res["us_certify_off"] = tim
print(json.dumps(res, indent=1))
json.dump(res, open("gpurun_out/gpu_err.json", "w"), indent=1)
