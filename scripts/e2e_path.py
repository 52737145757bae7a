"""nj_verify_host latency (host-resident q read in place) at B, gamma: alternating
between two Verifiers (NJ_HOSTQ_FUSED=1: the fused kernel up to 48 rows; 0: the
device-q rule, the staged step with the flat sampler above 24 rows).
usage: python scripts/e2e_path.py B gamma rounds"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_22420_b200 import Verifier  # noqa: E402
from synth.inputs import make_batch, make_weight  # noqa: E402

dev = torch.device("cuda:0")
V, d = 152064, 3584
B, g, rounds = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
W = make_weight(V, d, 1, dev)
b = make_batch(B, g, V=V, d=d, seed=3, device=dev, W=W)
vs = {}
for f in ("1", "0"):
    os.environ["NJ_HOSTQ_FUSED"] = f
    vs[f] = Verifier(d, V, max_batch=B, gamma_max=max(g, 1))
pin = lambda t: t.cpu().pin_memory()
hh, th, qh, uh = pin(b.hidden), pin(b.draft_tokens), pin(b.draft_probs), pin(b.uniforms)
ah = torch.empty(B, dtype=torch.int32).pin_memory()
nh = torch.empty(B, dtype=torch.int32).pin_memory()
res = {f: [] for f in vs}
outs = {}
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
        outs[f] = (ah.clone(), nh.clone())
assert (outs["1"][0] == outs["0"][0]).all() and (outs["1"][1] == outs["0"][1]).all()
for f, t in res.items():
    t.sort()
    m = t[len(t) // 2]
    print(f"B={B} g={g} NJ_HOSTQ_FUSED={f}: {m * 1e3:.1f} us per call (min {t[0] * 1e3:.1f} max {t[-1] * 1e3:.1f}), "
          f"{b.N / m * 1e3:.0f} positions/s", flush=True)
