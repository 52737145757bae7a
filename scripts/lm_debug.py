"""k_lmhead bring-up: logits of nj_lmhead_logits vs a torch fp32 matmul, per CTA-group / tile width."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_22420_b200 import Verifier  # noqa: E402

dev = torch.device("cuda:0")
cases = [(4096, 256, 100), (4096, 256, 256), (152064, 3584, 256), (152064, 3584, 400), (8192, 512, 300)]
for cg in (1, 2):
    os.environ["NJ_LM_CG"] = str(cg)
    for V, d, R in cases:
        g = torch.Generator(device=dev).manual_seed(R)
        W = (torch.randn(V, d, device=dev, generator=g) * 0.05).to(torch.bfloat16)
        h = torch.randn(R, d, device=dev, generator=g).to(torch.bfloat16)
        v = Verifier(d, V, max_batch=R, gamma_max=1)
        out = torch.full((R, V), float("nan"), device=dev)
        v.lmhead_logits(h, W, torch.arange(R, dtype=torch.int32, device=dev), out)
        torch.cuda.synchronize()
        ref = h.float() @ W.float().t()
        err = (out - ref).abs()
        bad = ~(err <= 1e-2)
        msg = f"cg={cg} V={V} d={d} R={R}: nan={int(torch.isnan(out).sum())} max_err={float(err.nan_to_num(1e9).max()):.3g}"
        if bad.any():
            rows = bad.any(1).nonzero().flatten()
            cols = bad.any(0).nonzero().flatten()
            msg += f" bad rows {int(rows.numel())} [{int(rows.min())}..{int(rows.max())}] cols {int(cols.numel())} [{int(cols.min())}..{int(cols.max())}]"
            r0 = int(rows[0])
            c0 = bad[r0].nonzero().flatten()[:8].tolist()
            msg += f" e.g. row {r0} cols {c0} got {out[r0, c0].tolist()[:4]} ref {ref[r0, c0].tolist()[:4]}"
        print(msg, flush=True)
        v.close()
