"""Per-kernel GPU time of nj_verify at the Qwen shape in an eager back-to-back loop
(NJ_LAUNCH_TIMES=1: libnj prints the per-kernel means at exit; device buffers only).
usage: NJ_LAUNCH_TIMES=1 python scripts/launch_times.py B gamma [steps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_22420_b200 import Verifier  # noqa: E402
from synth.inputs import make_batch, make_weight  # noqa: E402

dev = torch.device("cuda:0")
V, d = 152064, 3584
B, g = int(sys.argv[1]), int(sys.argv[2])
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
W = make_weight(V, d, 1, dev)
b = make_batch(B, g, V=V, d=d, seed=7, device=dev, W=W)
v = Verifier(d, V, max_batch=B, gamma_max=max(g, 1))
acc = torch.empty(B, dtype=torch.int32, device=dev)
nxt = torch.empty(B, dtype=torch.int32, device=dev)
for _ in range(steps):
    v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
torch.cuda.synchronize()
