"""Accuracy of the production GEMM vs the fp64 oracle for k_lmhead variants
(first accumulator group NJ_LM_KS0 k-blocks, the rest every 4) and k_gemm_big
(NJ_LM=0, restart every 4): per row |d ln p| over every entry with p > 1e-6,
|d lse|, and the max |F_gpu - F_ref| of the CDF of p (what an inverse-CDF draw
depends on).  Qwen shape, 256 rows (B=64, gamma=3 hidden states)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2512_22420_b200 import Verifier  # noqa: E402
from synth.inputs import make_batch, make_weight  # noqa: E402

dev = torch.device("cuda:0")
V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
W64 = oracle.weight_f64(oracle.bf16_bits(W))
b = make_batch(64, 3, V=V, d=d, seed=77, device=dev, W=W)
R = b.N
L = oracle.logits_blas(oracle.bf16_bits(b.hidden), None, W64=W64)
lse = np.logaddexp.reduce(L, axis=1)
P = np.exp(L - lse[:, None])
F = np.cumsum(P, axis=1)
res = {}
for name, env in [("gemm_big ks4", {"NJ_LM": "0"}), ("lmhead ks0=4", {"NJ_LM_KS0": "4"}),
                  ("lmhead ks0=8", {"NJ_LM_KS0": "8"}), ("lmhead ks0=12", {"NJ_LM_KS0": "12"}),
                  ("lmhead ks0=16", {"NJ_LM_KS0": "16"})]:
    for k in ("NJ_LM", "NJ_LM_KS0"):
        os.environ.pop(k, None)
    os.environ.update(env)
    v = Verifier(d, V, max_batch=R, gamma_max=1)
    out = torch.empty(R, V, device=dev)
    v.lmhead_logits(b.hidden, W, torch.arange(R, dtype=torch.int32, device=dev), out, ks=4)
    torch.cuda.synchronize()
    g = out.double().cpu().numpy()
    lg = np.logaddexp.reduce(g, axis=1)
    dlnp = np.abs((g - lg[:, None]) - (L - lse[:, None]))
    mask = (L - lse[:, None]) > np.log(1e-6)
    Fg = np.cumsum(np.exp(g - lg[:, None]), axis=1)
    dF = np.abs(Fg - F).max(axis=1)
    r = {"max_dlnp_p>1e-6": float(dlnp[mask].max()), "p99.99_dlnp": float(np.percentile(dlnp[mask], 99.99)),
         "max_dlse": float(np.abs(lg - lse).max()), "max_cdf_err": float(dF.max()),
         "median_cdf_err": float(np.median(dF))}
    res[name] = r
    print(name, json.dumps(r), flush=True)
    v.close()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/lm_accuracy.json", "w"), indent=1)
