"""nj_propose (0.5B-style head, d=896, V=151936, B=64) GEMM time under k_gemm_big knobs."""
import os, sys, json, torch
sys.path.insert(0, ".")
from paper_2512_22420_b200 import NJ_OPT_PROFILE, Verifier
from synth.inputs import make_batch, make_weight
dev = torch.device("cuda:0"); DV, DD = 151936, 896
W = make_weight(DV, DD, 9, dev)
KN = ["NJ_BIG_S", "NJ_BIG_GK", "NJ_BIG_MAXT", "NJ_BIG_NBUF", "NJ_TEAMS", "NJ_KS"]
out = {}
for B in (64, 256):
    b = make_batch(B, 0, V=DV, d=DD, seed=0, device=dev, W=W)
    for var in [{}, {"NJ_TEAMS": "0"}, {"NJ_BIG_GK": "2"}, {"NJ_BIG_GK": "7"}, {"NJ_BIG_NBUF": "4"}, {"NJ_BIG_MAXT": "32"},
                {"NJ_KS": "7"}, {"NJ_BIG_S": "2"}, {}]:
        for k in KN:
            os.environ.pop(k, None)
        os.environ.update(var)
        try:
            v = Verifier(DD, DV, max_batch=B, gamma_max=1)
            tok = torch.empty(B, dtype=torch.int32, device=dev); q = torch.empty(B, DV, device=dev)
            for _ in range(3): v.propose(b.hidden, W, b.uniforms, tok, q)
            torch.cuda.synchronize()
            v.set_option(NJ_OPT_PROFILE, 1); v.kernel_time(True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20): v.propose(b.hidden, W, b.uniforms, tok, q)
            e1.record(); torch.cuda.synchronize()
            kms, kn = v.kernel_time(True)
            r = (round(e0.elapsed_time(e1) / 20 * 1e3, 1), round(kms / kn * 1e3, 1))
            del v
        except Exception as e:
            r = str(e)[:100]
        key = f"B{B} " + (",".join(f"{k}={v_}" for k, v_ in var.items()) or "default")
        out[key] = r
        print(key, r, flush=True)
json.dump(out, open("gpurun_out/explore_propose.json", "w"), indent=1)
