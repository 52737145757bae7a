"""nj_verify_host latency at small N (host-resident q): the fused kernel vs the staged
step forced with NJ_OPT_PATH, alternating.  usage: python scripts/e2e_small_path.py B gamma rounds"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_22420_b200 import NJ_OPT_PATH, NJ_PATH_FUSED, NJ_PATH_STAGED, Verifier  # noqa: E402
from synth.inputs import make_batch, make_weight  # noqa: E402

dev = torch.device("cuda:0")
V, d = 152064, 3584
B, g, rounds = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
W = make_weight(V, d, 1, dev)
b = make_batch(B, g, V=V, d=d, seed=3, device=dev, W=W)
vs = {}
for name, path in (("fused", NJ_PATH_FUSED), ("staged", NJ_PATH_STAGED)):
    vs[name] = Verifier(d, V, max_batch=B, gamma_max=max(g, 1))
    vs[name].set_option(NJ_OPT_PATH, path)
pin = lambda t: t.cpu().pin_memory()
hh, th, qh, uh = pin(b.hidden), pin(b.draft_tokens), pin(b.draft_probs), pin(b.uniforms)
ah = torch.empty(B, dtype=torch.int32).pin_memory()
nh = torch.empty(B, dtype=torch.int32).pin_memory()
res = {f: [] for f in vs}
for r in range(rounds):
    for f, v in vs.items():
        for _ in range(2):
            v.verify_host(hh, W, th, qh, b.gamma, uh, ah, nh)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            v.verify_host(hh, W, th, qh, b.gamma, uh, ah, nh)
        e1.record()
        torch.cuda.synchronize()
        res[f].append(e0.elapsed_time(e1) / 20)
for f, t in res.items():
    t.sort()
    m = t[len(t) // 2]
    print(f"B={B} g={g} N={b.N} {f}: {m * 1e3:.1f} us per call, {b.N / m * 1e3:.0f} positions/s", flush=True)
