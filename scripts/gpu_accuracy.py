"""Tensor-core accumulation accuracy: rounding-mode microtests and error of
logits vs fresh-accumulator granularity ks (fp64 partial sums)."""
import json, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2512_22420_b200 import Verifier
from scripts.probes import _probe
from synth.inputs import make_batch, make_weight
dev = torch.device("cuda:0")
res = {}
# ---------------- rounding microtests (d = 32 -> 2 MMA steps of K=16)
def bf(x):
    return torch.tensor(x, dtype=torch.float32).to(torch.bfloat16)
d, V = 32, 16
cases = {
  "single_0.75ulp": ([1.0, 1.5 * 2**-24], []),
  "single_neg_0.75ulp": ([-1.0, -1.5 * 2**-24], []),
  "single_3x0.25ulp": ([1.0, 2**-25, 2**-25, 2**-25], []),
  "acc_0.75ulp": ([1.0], [1.5 * 2**-24]),
  "acc_neg_0.75ulp": ([-1.0], [-1.5 * 2**-24]),
  "acc_0.25ulp": ([1.0], [2**-25]),
}
W = torch.zeros(V, d, dtype=torch.bfloat16, device=dev)
names = list(cases)
for i, n in enumerate(names):
    a, b = cases[n]
    for k, x in enumerate(a): W[i, k] = bf(x)
    for k, x in enumerate(b): W[i, 16 + k] = bf(x)
h = torch.ones(1, d, dtype=torch.bfloat16, device=dev)
v = Verifier(d, V, max_batch=4, gamma_max=1)
out = torch.empty(1, V, device=dev)
v.lmhead_logits(h, W, torch.zeros(1, dtype=torch.int32, device=dev), out)
torch.cuda.synchronize()
exact = W.double().sum(1)
ulp = 2.0**-23
res["rounding"] = {n: {"exact_minus_1_in_ulp": float((exact[i].abs() - 1) / ulp),
                       "tc_minus_1_in_ulp": float((out[0, i].double().abs() - 1) / ulp)} for i, n in enumerate(names)}
del v
# ---------------- accuracy vs ks at the C2 shape
V, d = 152064, 3584
Wf = make_weight(V, d, 0, dev)
b = make_batch(8, 3, V=V, d=d, seed=11, device=dev, W=Wf)
R = b.N
rows = torch.arange(R, dtype=torch.int32, device=dev)
Ld = b.hidden.double() @ Wf.double().t()
Pd = torch.softmax(Ld, 1); Fd = torch.cumsum(Pd, 1); lse_d = torch.logsumexp(Ld, 1)
v = Verifier(d, V, max_batch=64, gamma_max=5)
def stats(L):
    dl = L - Ld
    ks_, rs = [], []
    for r in range(R):
        x = Ld[r]; y = dl[r]
        A = torch.stack([torch.ones_like(x), x], 1)
        sol = torch.linalg.lstsq(A, y[:, None]).solution[:, 0]
        ks_.append(float(sol[1])); rs.append(float((y - A @ sol).std()))
    P = torch.softmax(L, 1)
    F = torch.cumsum(P, 1)
    top = Pd.argmax(1)
    return {"kappa": float(np.mean(ks_)), "resid_std": float(np.mean(rs)), "dl_max": float(dl.abs().max()),
            "lse_err": float((torch.logsumexp(L, 1) - lse_d).abs().max()),
            "F_err_max": float((F - Fd).abs().max()), "F_err_mean": float((F - Fd).abs().mean()),
            "lnp_err_max_p>1e-3": float(((torch.log(P) - torch.log(Pd)).abs() * (Pd > 1e-3)).max())}
L32 = torch.empty(R, V, device=dev)
v.lmhead_logits(b.hidden, Wf, rows, L32); torch.cuda.synchronize()
res["plain"] = stats(L32.double())
for ks in [1, 2, 4, 8, 16, 56, 224]:
    L = torch.empty(R, V, dtype=torch.float64, device=dev)
    _probe.logits_ks(b.hidden[rows.long()], Wf, L, ks)
    torch.cuda.synchronize()
    st = stats(L)
    st["f32_rounded"] = stats(L.float().double())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        _probe.logits_ks(b.hidden[rows.long()], Wf, L, ks)
    e1.record(); torch.cuda.synchronize()
    st["us"] = e0.elapsed_time(e1) / 5 * 1e3
    res[f"ks{ks}"] = st
    print(ks, json.dumps(st), flush=True)
print(json.dumps(res, indent=1))
json.dump(res, open("gpurun_out/gpu_accuracy.json", "w"), indent=1)
