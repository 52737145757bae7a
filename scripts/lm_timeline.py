"""k_lmhead timeline of CTA 0 (NJ_PHASE_TS=1): per ring stage the producer's wait
for a free slot and the MMA warp's wait for operands / issue+commit, for the
given probe bits (NJ_LM_DBG) at R rows.  usage: lm_timeline.py R DBG[,DBG...]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["NJ_PHASE_TS"] = "1"
from paper_2512_22420_b200 import Verifier, load  # noqa: E402

lib = load()
lib.nj_debug_phase_times.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
dev = torch.device("cuda:0")
V, d = 152064, 3584
R = int(sys.argv[1])
g = torch.Generator(device=dev).manual_seed(0)
W = (torch.randn(V, d, device=dev, generator=g) * 0.05).to(torch.bfloat16)
h = torch.randn(R, d, device=dev, generator=g).to(torch.bfloat16)
out = torch.empty(R, V, device=dev)
for dbg in sys.argv[2].split(","):
    for kv in dbg.split(";"):
        k, val = kv.split("=") if "=" in kv else ("NJ_LM_DBG", kv)
        os.environ[k] = val
    mb = min(R, 768)
    v = Verifier(d, V, max_batch=mb, gamma_max=(R + mb - 1) // mb)
    rows = torch.arange(R, dtype=torch.int32, device=dev)
    for _ in range(3):
        v.lmhead_logits(h, W, rows, out)
    torch.cuda.synchronize()
    ts = np.zeros(20 * 1024, np.uint64)
    lib.nj_debug_phase_times(v._h, ts.ctypes.data, 20 * 1024)
    t = ts.astype(np.int64)
    P = t[:4000].reshape(2000, 2)
    M = t[4096:4096 + 3 * 1300].reshape(1300, 3)
    M = M[M[:, 0] > 0]          # (MB > 1 stamps every MB-th stage)
    P = P[P[:, 0] > 0]
    n = min(len(M), len(P))
    M = M[:n]
    P = P[:n]
    t0 = M[0, 0]
    per = np.diff(M[:, 0])
    print(f"dbg={dbg} R={R}: stages {n}, per stage median {np.median(per):.0f} ns (p10 {np.percentile(per, 10):.0f}, "
          f"p90 {np.percentile(per, 90):.0f}); MMA wait-full median {np.median(M[:, 1] - M[:, 0]):.0f} ns, "
          f"issue+commit {np.median(M[:, 2] - M[:, 1]):.0f} ns; producer wait-empty median "
          f"{np.median(P[:, 1] - P[:, 0]):.0f} ns, producer per stage {np.median(np.diff(P[:, 0])):.0f} ns", flush=True)
    span = M[-1, 2] - M[0, 0]
    wf = M[:, 1] - M[:, 0]
    ic = M[:, 2] - M[:, 1]
    print(f"   mean per stage {span / (n - 1):.0f} ns; mean wait-full {wf.mean():.0f} (>500ns: {int((wf > 500).sum())} stages, "
          f"{wf[wf > 500].sum() / span * 100:.1f} % of span); mean issue+commit {ic.mean():.0f} (>500ns: "
          f"{int((ic > 500).sum())}, {ic[ic > 500].sum() / span * 100:.1f} % of span); gaps {((M[1:, 0] - M[:-1, 2]).mean()):.0f}")
    O = t[8192:8192 + 4000].reshape(2000, 2)[:1900]
    O = O[O[:, 0] > 0]
    if len(O):
        od = O[:, 1] - O[:, 0]
        print(f"   items {len(O)}: output median {np.median(od):.0f} ns mean {od.mean():.0f}; item period "
              f"{np.median(np.diff(O[:, 0])) if len(O) > 1 else 0:.0f} ns")
    Gs = t[12288:12288 + 2000].reshape(1000, 2)
    ng = int((Gs[:, 0] > 0).sum())
    Gs = Gs[:ng]
    A = t[14336:14336 + ng]
    if ng > 2:
        wait = Gs[:, 1] - Gs[:, 0]
        drain = A - Gs[:len(A), 1]
        print(f"   epilogue warp0 groups {ng}: afull wait median {np.median(wait):.0f} ns mean {wait.mean():.0f}; "
              f"drain (wait end -> arrive) median {np.median(drain):.0f} ns mean {drain.mean():.0f}; group period "
              f"{np.median(np.diff(Gs[:, 1])):.0f} ns")
    AE = t[16384:16384 + 2000].reshape(1000, 2)
    na = int((AE[:, 0] > 0).sum())
    if na > 2:
        AE = AE[:na]
        aw = AE[:, 1] - AE[:, 0]
        ngi = int(os.environ.get("NGROUPS", "14"))
        first = aw[0::ngi]
        rest = np.delete(aw, np.s_[0::ngi])
        span_a = AE[-1, 1] - AE[0, 0]
        print(f"   MMA aempty waits {na}: total {aw.sum() / span_a * 100:.1f} % of span; first group of an item "
              f"median {np.median(first):.0f} ns mean {first.mean():.0f}; other groups median {np.median(rest):.0f} "
              f"mean {rest.mean():.0f} ns; sum first {first.sum() / span_a * 100:.1f} %, rest {rest.sum() / span_a * 100:.1f} %")
    # first 12 stages raw (relative ns)
    print("   MMA  ", [(int(a - t0), int(b - t0), int(c - t0)) for a, b, c in M[20:28]])
    print("   prod ", [(int(a - t0), int(b - t0)) for a, b in P[20:28]])
    v.close()
