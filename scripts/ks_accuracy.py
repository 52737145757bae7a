"""Accuracy of the production GEMM (k_gemm_big via nj_lmhead_logits) vs the
accumulator restart period ks (k-blocks): |d ln p| over every vocabulary entry
with p > 1e-6 and at the drafted tokens, Qwen shape, 256 rows vs the fp64
oracle.  Sets the acceptance certificates of DESIGN.md §6."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
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
res = {}
v = Verifier(d, V, max_batch=R, gamma_max=1)
for ks in (4, 8, 14, 28, 56):
    out = torch.empty(R, V, device=dev)
    v.lmhead_logits(b.hidden, W, torch.arange(R, dtype=torch.int32, device=dev), out, ks=ks)
    torch.cuda.synchronize()
    g = out.double().cpu().numpy()
    lg = np.logaddexp.reduce(g, axis=1)
    dlnp = np.abs((g - lg[:, None]) - (L - lse[:, None]))
    mask = (L - lse[:, None]) > np.log(1e-6)
    r = {"max_dlnp_p>1e-6": float(dlnp[mask].max()), "p99.99_dlnp": float(np.percentile(dlnp[mask], 99.99)),
         "max_dl": float(np.abs(g - L).max()), "max_dlse": float(np.abs(lg - lse).max())}
    res[ks] = r
    print(ks, json.dumps(r), flush=True)
json.dump(res, open("gpurun_out/ks_accuracy.json", "w"), indent=1)
