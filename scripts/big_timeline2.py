"""Where the MMA thread and the epilogue of k_gemm_big CTA 0 wait (NJ_PHASE_TS):
per stage: MMA wait-for-data, issue+commit; per group: MMA wait-for-drained
accumulator; epilogue wait-for-accumulator and drain time."""
import ctypes, os, sys, numpy as np, torch
sys.path.insert(0, ".")
os.environ["NJ_PHASE_TS"] = "1"
from paper_2512_22420_b200 import NJ_OPT_CERTIFY, Verifier, load
from synth.inputs import make_batch, make_weight
lib = load(); lib.nj_debug_phase_times.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
dev = torch.device("cuda:0"); V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
for B, g, extra in [(64, 3, {}), (16, 3, {})]:
    for k in ("NJ_KS",):
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
    M = t[4096:4096 + 3 * 1300].reshape(1300, 3)
    M = M[M[:, 0] > 0]
    E = t[8192:8192 + 4096].reshape(2048, 2)
    E = E[E[:, 0] > 0]
    A = t[12288:12288 + 4000].reshape(2000, 2)
    A = A[A[:, 0] > 0]
    span = (M[-1, 2] - M[0, 0]) / 1e3
    print(f"== B={B} g={g} {extra}: {len(M)} stages in {span:.1f} us ({span * 1e3 / len(M):.0f} ns/stage)")
    wf = M[:, 1] - M[:, 0]; iss = M[:, 2] - M[:, 1]; gap = M[1:, 0] - M[:-1, 2]
    print("  MMA wait full   ns: mean %.0f median %.0f  (sum %.1f us)" % (wf.mean(), np.median(wf), wf.sum() / 1e3))
    print("  MMA issue+commit ns: mean %.0f median %.0f  (sum %.1f us)" % (iss.mean(), np.median(iss), iss.sum() / 1e3))
    print("  MMA loop gap    ns: mean %.0f median %.0f  (sum %.1f us, incl. aempty waits)" % (gap.mean(), np.median(gap), gap.sum() / 1e3))
    wa = A[:, 1] - A[:, 0]
    print("  MMA wait aempty ns: mean %.0f median %.0f  (sum %.1f us over %d groups)" % (wa.mean(), np.median(wa), wa.sum() / 1e3, len(A)))
    we = E[1:, 0] - E[:-1, 1]
    dr = E[:, 1] - E[:, 0]
    print("  EPI wait+drain per group ns: mean %.0f median %.0f ; between groups (item work) mean %.0f median %.0f max %.0f" % (
        dr.mean(), np.median(dr), we.mean(), np.median(we), we.max()))
    del v
