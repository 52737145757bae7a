"""Per-item epilogue output timing of k_gemm_big CTA 0, warp 2 (NJ_PHASE_TS):
logits/capture section and stats section, per item."""
import ctypes, os, sys, numpy as np, torch
sys.path.insert(0, ".")
os.environ["NJ_PHASE_TS"] = "1"
from paper_2512_22420_b200 import NJ_OPT_CERTIFY, Verifier, load
from synth.inputs import make_batch, make_weight
lib = load(); lib.nj_debug_phase_times.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
dev = torch.device("cuda:0"); V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
for (B, g, sm) in [(64, 3, "0"), (64, 3, "1"), (256, 5, "0"), (256, 5, "1")]:
    os.environ["NJ_STATS"] = sm
    b = make_batch(B, g, V=V, d=d, seed=0, device=dev, W=W)
    v = Verifier(d, V, max_batch=B, gamma_max=5); v.set_option(NJ_OPT_CERTIFY, 0)
    acc = torch.empty(B, dtype=torch.int32, device=dev); nxt = torch.empty(B, dtype=torch.int32, device=dev)
    for _ in range(3): v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
    torch.cuda.synchronize()
    ts = np.zeros(16 * 1024, np.uint64)
    lib.nj_debug_phase_times(v._h, ts.ctypes.data, 16 * 1024)
    t = ts.astype(np.int64)[14336:14336 + 2000].reshape(500, 4)
    t = t[(t[:, 0] > 0) & (t[:, 2] > 0)]
    wr = t[:, 1] - t[:, 0]; st = t[:, 2] - t[:, 1]
    print(f"B={B} g={g} stats_mode={sm}: items {len(t)}  logits+capture ns median {np.median(wr):.0f}  stats ns median {np.median(st):.0f} max {st.max():.0f}")
    del v
