"""Dominant-kernel (k_gemm_big / k_fused_verify) and step time under knob
variants (env, read at nj_create), certificate off.  usage:
  python scripts/explore_knobs.py '<json list of (B, gamma)>' '<json list of env dicts>'"""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_22420_b200 import NJ_OPT_CERTIFY, NJ_OPT_PROFILE, Verifier  # noqa: E402
from synth.inputs import make_batch, make_weight  # noqa: E402

dev = torch.device("cuda:0")
V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
points = json.loads(sys.argv[1])
variants = json.loads(sys.argv[2])
allk = sorted({k for v in variants for k in v})
for B, g in points:
    b = make_batch(B, g, V=V, d=d, seed=5, device=dev, W=W)
    for var in variants:
        for k in allk:
            os.environ.pop(k, None)
        os.environ.update(var)
        try:
            v = Verifier(d, V, max_batch=B, gamma_max=5)
            v.set_option(NJ_OPT_CERTIFY, 0)
            acc = torch.empty(B, dtype=torch.int32, device=dev)
            nxt = torch.empty(B, dtype=torch.int32, device=dev)
            for _ in range(3):
                v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
            torch.cuda.synchronize()
            v.set_option(NJ_OPT_PROFILE, 1)
            v.kernel_time(True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
            e1.record()
            torch.cuda.synchronize()
            kms, kn = v.kernel_time(True)
            r = {"step_us": round(e0.elapsed_time(e1) / 10 * 1e3, 1), "kernel_us": round(kms / kn * 1e3, 1)}
            del v
        except Exception as ex:
            r = {"error": str(ex)[:120]}
        print(json.dumps({"B": B, "gamma": g, "knobs": var, **r}), flush=True)
