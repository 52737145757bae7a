"""nj_verify_host latency at the C2 shape vs the number of staged q rows
(NJ_OPT_Q_STAGE_ROWS), plus the raw pinned-host -> device copy bandwidth.
usage: python scripts/e2e_qstage.py [B] [gamma]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_22420_b200 import NJ_OPT_Q_STAGE_ROWS, Verifier  # noqa: E402
from synth.inputs import make_batch, make_weight  # noqa: E402

dev = torch.device("cuda:0")
V, d = 152064, 3584
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
g = int(sys.argv[2]) if len(sys.argv) > 2 else 3
for mb in (0.6, 8, 32):
    n = int(mb * 2**20 / 4)
    h = torch.empty(n).pin_memory()
    dd = torch.empty(n, device=dev)
    for _ in range(3):
        dd.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        dd.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10
    print(f"H2D pinned {mb:5.1f} MB: {t * 1e3:8.1f} us  {n * 4 / t / 1e6:6.1f} GB/s", flush=True)
W = make_weight(V, d, 1, dev)
b = make_batch(B, g, V=V, d=d, seed=3, device=dev, W=W)
v = Verifier(d, V, max_batch=B, gamma_max=max(g, 1))
pin = lambda t: t.cpu().pin_memory()
hh, th, qh, uh = pin(b.hidden), pin(b.draft_tokens), pin(b.draft_probs), pin(b.uniforms)
ah = torch.empty(B, dtype=torch.int32).pin_memory()
nh = torch.empty(B, dtype=torch.int32).pin_memory()
for nst in (0, 1, 4, 8, 13, 24, -1):
    v.set_option(NJ_OPT_Q_STAGE_ROWS, nst)
    for _ in range(3):
        v.verify_host(hh, W, th, qh, b.gamma, uh, ah, nh)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        v.verify_host(hh, W, th, qh, b.gamma, uh, ah, nh)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 20
    print(f"stage rows {nst:3d} (staged {len(v.host_staged_rows()):3d}): {t * 1e3:7.1f} us per call, "
          f"{b.N / t * 1e3:8.0f} positions/s; path {v.plan(b.gamma)[0]}", flush=True)
