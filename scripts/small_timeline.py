"""Phase timeline of the C2 staged step (NJ_PHASE_TS=1): k_lmhead's per-CTA end
stamps and k_sample_small's per-CTA phase stamps, relative to the last k_lmhead
CTA's end.  usage: python scripts/small_timeline.py [B] [gamma] [reps]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["NJ_PHASE_TS"] = "1"
from paper_2512_22420_b200 import Verifier, load  # noqa: E402
from synth.inputs import make_batch, make_weight  # noqa: E402

lib = load()
lib.nj_debug_phase_times.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
dev = torch.device("cuda:0")
V, d = 152064, 3584
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
g = int(sys.argv[2]) if len(sys.argv) > 2 else 3
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
W = make_weight(V, d, 1, dev)
v = Verifier(d, V, max_batch=B, gamma_max=max(g, 1))
names = ["start", "wait done", "row lse", "acceptance", "chunk masses", "cluster sync 1", "gather + sync 2",
         "prefix done", "token written"]
rows = []
for r in range(reps + 2):
    b = make_batch(B, g, V=V, d=d, seed=100 + r, device=dev, W=W)
    acc = torch.empty(B, dtype=torch.int32, device=dev)
    nxt = torch.empty(B, dtype=torch.int32, device=dev)
    v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
    torch.cuda.synchronize()
    ts = np.zeros(24 * 1024, np.uint64)
    lib.nj_debug_phase_times(v._h, ts.ctypes.data, 24 * 1024)
    t = ts.astype(np.int64)
    lm_end = t[20480:20480 + 512]
    lm_end = lm_end[lm_end > 0]
    S = t[18432:18432 + 2048].reshape(128, 16)[:, :9]
    if r < 2 or len(lm_end) == 0:
        continue
    t0 = lm_end.max()
    act = S[:, 0] > 0
    rel = np.where(S > 0, S - t0, np.nan)[act]
    rows.append((lm_end.min() - t0, rel))
    print(f"rep {r}: k_lmhead CTA ends span {(lm_end.max() - lm_end.min()) / 1e3:.1f} us; sampler CTAs {act.sum()}")
    for k, n in enumerate(names):
        col = rel[:, k]
        col = col[~np.isnan(col)]
        if len(col):
            print(f"   {n:16s} median {np.median(col) / 1e3:7.2f} us  min {col.min() / 1e3:7.2f}  max {col.max() / 1e3:7.2f}  (n={len(col)})")
