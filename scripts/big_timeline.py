"""Per-stage timeline of k_gemm_big CTA 0 (NJ_PHASE_TS=1): producer / MMA stage
start times and epilogue group completions (globaltimer, ns)."""
import ctypes, os, sys, numpy as np, torch
sys.path.insert(0, ".")
os.environ["NJ_PHASE_TS"] = "1"
from paper_2512_22420_b200 import NJ_OPT_CERTIFY, Verifier, load
from synth.inputs import make_batch, make_weight
lib = load(); lib.nj_debug_phase_times.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
dev = torch.device("cuda:0"); V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
VARS = [(64, 3, {"NJ_BIG_DBG": "15", "NJ_BIG_S": str(S)}) for S in (2, 4, 8, 16, 32)] + [(64, 3, {"NJ_BIG_DBG": "15", "NJ_BIG_S": "16", "NJ_KS": "56"})]
for B, g, extra in VARS:
    for k in ("NJ_BIG_DBG", "NJ_BIG_S", "NJ_KS"):
        os.environ.pop(k, None)
    os.environ.update(extra)
    b = make_batch(B, g, V=V, d=d, seed=0, device=dev, W=W)
    v = Verifier(d, V, max_batch=B, gamma_max=5); v.set_option(NJ_OPT_CERTIFY, 0)
    acc = torch.empty(B, dtype=torch.int32, device=dev); nxt = torch.empty(B, dtype=torch.int32, device=dev)
    for _ in range(3): v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
    torch.cuda.synchronize()
    ts = np.zeros(16 * 1024, np.uint64)
    lib.nj_debug_phase_times(v._h, ts.ctypes.data, 16 * 1024)
    t = ts.astype(np.int64)
    P, M, E = t[:4096], t[4096:8192], t[8192:12288]
    n = int((P > 0).sum()); nm = int((M > 0).sum()); ne = int((E > 0).sum())
    t0 = P[0]
    print(f"== B={B} g={g} {extra}: stages {n} (mma {nm}), groups {ne}, total {(max(P[n-1], M[nm-1], E[ne-1]) - t0)/1e3:.1f} us")
    dP = np.diff(P[:n]); dM = np.diff(M[:nm]); dE = np.diff(E[:ne])
    print("  producer stage interval ns: median %.0f p90 %.0f max %.0f" % (np.median(dP), np.percentile(dP, 90), dP.max()))
    print("  mma stage interval ns:      median %.0f p90 %.0f max %.0f" % (np.median(dM), np.percentile(dM, 90), dM.max()))
    print("  epilogue group interval ns: median %.0f p90 %.0f max %.0f" % (np.median(dE), np.percentile(dE, 90), dE.max()))
    print("  mma start - producer start (same stage) ns: median %.0f" % np.median(M[:min(n, nm)] - P[:min(n, nm)]))
    print("  first 30 mma intervals:", dM[:30].tolist())
    del v
