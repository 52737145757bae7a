"""C2 (fused path) step time under the fused kernel's knobs (read at
nj_create): k-blocks per ring stage (NJ_KGROUP), scratch groups (NJ_FGROUPS).
CUDA-graph replays, 4 rotating batches, median of 5 x 50 steps."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2512_22420_b200 import Verifier  # noqa: E402
from synth.inputs import make_batch, make_weight  # noqa: E402

dev = torch.device("cuda:0")
V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
bs = [make_batch(8, 3, V=V, d=d, seed=100 + i, device=dev, W=W) for i in range(4)]
KN = ["NJ_KGROUP", "NJ_FGROUPS", "NJ_SACC", "NJ_KPD"]
res = []
for var in json.loads(sys.argv[1]) if len(sys.argv) > 1 else [{}, {"NJ_KGROUP": "3"}, {"NJ_KGROUP": "2"}]:
    for k in KN:
        os.environ.pop(k, None)
    os.environ.update(var)
    v = Verifier(d, V, max_batch=8, gamma_max=5)
    acc = torch.empty(8, dtype=torch.int32, device=dev)
    nxt = torch.empty(8, dtype=torch.int32, device=dev)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    gs = []
    with torch.cuda.stream(s):
        for b in bs:
            v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
        s.synchronize()
        for b in bs:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
            gs.append(g)
    torch.cuda.current_stream().wait_stream(s)
    ts = []
    for rep in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(50):
            gs[i % 4].replay()
        e1.record()
        torch.cuda.synchronize()
        if rep:
            ts.append(e0.elapsed_time(e1) / 50 * 1e3)
    r = {"knobs": var, "us_median": float(np.median(ts)), "us_min": float(min(ts))}
    res.append(r)
    print(json.dumps(r), flush=True)
    del gs, v
