"""k_gemm_big timeline of CTA 0 (NJ_PHASE_TS=1): per ring stage the MMA warp's
wait-for-operands and issue+commit time, per accumulator group its wait for a
drained buffer, per group the epilogue's wait+drain, and per item the output
time -- for the full kernel and the handshake skeleton (NJ_BIG_DBG=15)."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
os.environ["NJ_PHASE_TS"] = "1"
from paper_2512_22420_b200 import NJ_OPT_CERTIFY, Verifier, load  # noqa: E402
from synth.inputs import make_batch, make_weight  # noqa: E402

lib = load()
lib.nj_debug_phase_times.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
dev = torch.device("cuda:0")
V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
out = []
for B, g in [(64, 3), (256, 5)]:
    for dbg in ["0", "15"]:
        os.environ["NJ_BIG_DBG"] = dbg
        b = make_batch(B, g, V=V, d=d, seed=0, device=dev, W=W)
        v = Verifier(d, V, max_batch=B, gamma_max=5)
        v.set_option(NJ_OPT_CERTIFY, 0)
        acc = torch.empty(B, dtype=torch.int32, device=dev)
        nxt = torch.empty(B, dtype=torch.int32, device=dev)
        for _ in range(3):
            v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
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
        I = t[14336:14336 + 2000].reshape(500, 4)
        I = I[I[:, 0] > 0]
        r = {"B": B, "gamma": g, "dbg": dbg, "stages": int(len(M)), "groups": int(len(A))}
        if len(M) > 2:
            span = (M[-1, 2] - M[0, 0]) / 1e3
            r["mma_span_us"] = span
            r["ns_per_stage"] = span * 1e3 / len(M)
            r["mma_wait_full_ns_median"] = float(np.median(M[:, 1] - M[:, 0]))
            r["mma_issue_commit_ns_median"] = float(np.median(M[:, 2] - M[:, 1]))
            r["mma_wait_full_us_sum"] = float((M[:, 1] - M[:, 0]).sum() / 1e3)
            r["mma_issue_us_sum"] = float((M[:, 2] - M[:, 1]).sum() / 1e3)
        if len(A):
            wa = A[:, 1] - A[:, 0]
            r["mma_wait_aempty_ns_median"] = float(np.median(wa))
            r["mma_wait_aempty_us_sum"] = float(wa.sum() / 1e3)
        if len(E) > 1:
            dr = E[:, 1] - E[:, 0]
            r["epi_wait_drain_ns_median"] = float(np.median(dr))
            gaps = E[1:, 0] - E[:-1, 1]
            r["epi_between_groups_ns_median"] = float(np.median(gaps))
            r["epi_between_groups_ns_max"] = float(gaps.max())
        if len(I):
            r["item_output_ns_median"] = float(np.median(I[:, 1] - I[:, 0]) + np.median(I[:, 2] - I[:, 1]))
        out.append(r)
        print(json.dumps(r), flush=True)
        del v
json.dump(out, open("gpurun_out/big_timeline4.json", "w"), indent=1)
