"""Per-phase timeline of k_fused_verify at C2 (B=8, gamma=3; NJ_PHASE_TS=1):
stamp k of every CTA (globaltimer ns), reported relative to the earliest
stamp 0, as median / max over CTAs.  Stamps: 0 start, 1 GEMM done, 2 after
barrier 1, 3 lse partials loaded, 4 lse, 5 acceptance / first rejection,
6 q slices, 7 masses, 8 CTA mass stored, 9 after barrier 2, 11 owner located,
12 draw done."""
import ctypes, os, sys, numpy as np, torch
sys.path.insert(0, ".")
os.environ["NJ_PHASE_TS"] = "1"
from paper_2512_22420_b200 import NJ_OPT_CERTIFY, Verifier, load
from synth.inputs import make_batch, make_weight
lib = load(); lib.nj_debug_phase_times.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
dev = torch.device("cuda:0"); V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
for B, g in [(8, 3), (1, 0), (12, 3)]:
    b = make_batch(B, g, V=V, d=d, seed=0, device=dev, W=W)
    v = Verifier(d, V, max_batch=B, gamma_max=5); v.set_option(NJ_OPT_CERTIFY, 1)
    acc = torch.empty(B, dtype=torch.int32, device=dev); nxt = torch.empty(B, dtype=torch.int32, device=dev)
    rows = []
    for rep in range(6):
        v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
        torch.cuda.synchronize()
        ts = np.zeros(16 * 1024, np.uint64)
        lib.nj_debug_phase_times(v._h, ts.ctypes.data, 16 * 1024)
        t = ts.astype(np.int64).reshape(-1, 16)
        t = t[t[:, 0] > 0]
        if rep >= 2:
            rows.append(t)
    print(f"== B={B} gamma={g}: {rows[0].shape[0]} CTAs")
    for k in [1, 2, 3, 4, 5, 6, 7, 8, 9, 11, 12]:
        med = np.median([np.median(t[:, k] - t[:, 0].min()) for t in rows]) / 1e3
        mx = np.median([np.max(t[:, k] - t[:, 0].min()) for t in rows]) / 1e3
        print(f"  stamp {k:2d}: median {med:8.2f} us   max {mx:8.2f} us")
    del v
