"""k_lmhead bring-up: staged-path debug outputs (lse, p_draft, flags) at the Qwen shape per CTA group."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_22420_b200 import NJ_OPT_PATH, NJ_PATH_STAGED, Verifier  # noqa: E402
from synth.inputs import make_batch, make_weight  # noqa: E402

dev = torch.device("cuda:0")
W = make_weight(152064, 3584, 0, dev)
for B, g in [(100, 3), (64, 3), (30, 3)]:
    b = make_batch(B, g, V=152064, d=3584, seed=32, device=dev, W=W)
    for env in ({"NJ_LM": "0"}, {"NJ_LM_CG": "1"}, {"NJ_LM_CG": "2"}):
        for k in ("NJ_LM", "NJ_LM_CG"):
            os.environ.pop(k, None)
        os.environ.update(env)
        v = Verifier(3584, 152064, max_batch=B, gamma_max=5)
        v.set_option(NJ_OPT_PATH, NJ_PATH_STAGED)
        acc = torch.zeros(B, dtype=torch.int32, device=dev)
        nxt = torch.zeros(B, dtype=torch.int32, device=dev)
        dd = {"lse": torch.full((b.N,), float("nan"), device=dev), "p_draft": torch.zeros(b.G, device=dev),
              "mass": torch.zeros(B, dtype=torch.float64, device=dev), "flags": torch.zeros(B, dtype=torch.int32, device=dev)}
        v.verify(b.hidden, b.W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt, debug=dd)
        torch.cuda.synchronize()
        print(B, g, env, "lse", dd["lse"][:5].tolist(), "pd", dd["p_draft"][:4].tolist(), "flags",
              int((dd["flags"] != 0).sum()), "nan pd", int(torch.isnan(dd["p_draft"]).sum()), flush=True)
        v.close()
