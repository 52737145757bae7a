"""Interleaved A/B timing of the production LM-head GEMM (nj_lmhead_logits -> k_lmhead)
under several knob sets: one Verifier per knob set (knobs are read at nj_create), the
sets timed round-robin so that the power-capped SM clock drifts equally over all of
them.  Reports the median µs per launch of each set over the rounds.

usage: python scripts/ab_lm.py R[,R...] ROUNDS 'K=V;K=V' 'K=V' ...   ('' = defaults)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_22420_b200 import Verifier  # noqa: E402

V, d = 152064, 3584
dev = torch.device("cuda:0")
Rs = [int(x) for x in sys.argv[1].split(",")]
rounds = int(sys.argv[2])
combos = sys.argv[3:] or [""]
g = torch.Generator(device=dev).manual_seed(0)
W = (torch.randn(V, d, device=dev, generator=g) * 0.05).to(torch.bfloat16)
Rmax = max(Rs)
h = torch.randn(Rmax, d, device=dev, generator=g).to(torch.bfloat16)
out = torch.empty(Rmax, V, device=dev)
for R in Rs:
    vs = []
    for combo in combos:
        env = dict(kv.split("=") for kv in combo.split(";") if kv)
        saved = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        mb = min(R, 768)
        vs.append(Verifier(d, V, max_batch=mb, gamma_max=(R + mb - 1) // mb))
        for k, val in saved.items():
            if val is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = val
    rows = torch.arange(R, dtype=torch.int32, device=dev)
    ref = None
    for i, v in enumerate(vs):
        for _ in range(2):
            v.lmhead_logits(h, W, rows, out[:R])
        torch.cuda.synchronize()
        if i == 0:
            ref = out[:R].clone()
        else:
            err = (out[:R] - ref).abs().max().item()
            if err > 1e-3:
                print(f"  !! {combos[i]!r} differs from {combos[0]!r} by {err:.3g}", flush=True)
    ts = [[] for _ in vs]
    reps = max(3, int(20000 / (R + 256)))
    for _ in range(rounds):
        for i, v in enumerate(vs):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                v.lmhead_logits(h, W, rows, out[:R])
            e1.record()
            torch.cuda.synchronize()
            ts[i].append(e0.elapsed_time(e1) * 1e3 / reps)
    fl = 2.0 * R * V * d
    for combo, t in zip(combos, ts):
        t.sort()
        m = t[len(t) // 2]
        print(f"R={R:5d} {combo or 'default':40s} {m:8.1f} us (min {t[0]:.1f} max {t[-1]:.1f})  "
              f"{fl / m / 1e6:7.1f} TF/s", flush=True)
    for v in vs:
        v.close()
