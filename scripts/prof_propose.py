import sys, torch
sys.path.insert(0, ".")
from paper_2512_22420_b200 import Verifier
from synth.inputs import make_batch, make_weight
dev = torch.device("cuda:0"); DV, DD, B = 151936, 896, int(sys.argv[1]) if len(sys.argv) > 1 else 64
W = make_weight(DV, DD, 9, dev)
b = make_batch(B, 0, V=DV, d=DD, seed=0, device=dev, W=W)
v = Verifier(DD, DV, max_batch=B, gamma_max=1)
tok = torch.empty(B, dtype=torch.int32, device=dev); q = torch.empty(B, DV, device=dev)
for _ in range(4):
    v.propose(b.hidden, W, b.uniforms, tok, q)
torch.cuda.synchronize()
