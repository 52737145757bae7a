import sys, torch
sys.path.insert(0, ".")
from paper_2512_22420_b200 import NJ_OPT_PATH, NJ_PATH_FUSED, NJ_PATH_TWOPASS, NJ_OPT_CERTIFY, Verifier
from synth.inputs import make_batch, make_weight
dev = torch.device("cuda:0")
V, d = 152064, 3584
B, g = int(sys.argv[1]), int(sys.argv[2])
path = {"fused": 1, "twopass": 2, "staged": 3}[sys.argv[3] if len(sys.argv) > 3 else "fused"]
W = make_weight(V, d, 0, dev)
b = make_batch(B, g, V=V, d=d, seed=0, device=dev, W=W)
v = Verifier(d, V, max_batch=B, gamma_max=5)
v.set_option(NJ_OPT_PATH, path)
acc = torch.empty(B, dtype=torch.int32, device=dev); nxt = torch.empty(B, dtype=torch.int32, device=dev)
for _ in range(4):
    v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
torch.cuda.synchronize()
