"""First-light GPU validation (run under gpurun): GEMM probe vs torch fp32,
fused / two-pass nj_verify vs the fp64 oracle, rough timings.  Each stage is
isolated so one failure does not hide the others."""
import json
import sys
import time
import traceback

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402  (test infrastructure)
from paper_2512_22420_b200 import NJ_OPT_PATH, NJ_PATH_FUSED, NJ_PATH_TWOPASS, Verifier  # noqa: E402
from synth.inputs import make_batch, make_weight  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda:0")
out = {}


SEL = sys.argv[1:]


def stage(name):
    def deco(f):
        if SEL and name not in SEL:
            return f
        t = time.time()
        try:
            r = f()
            out[name] = {"ok": True, **(r or {}), "s": round(time.time() - t, 2)}
        except Exception as e:  # noqa: BLE001
            out[name] = {"ok": False, "err": repr(e), "tb": traceback.format_exc()[-1500:]}
        print(name, json.dumps(out[name])[:2000], flush=True)
        return f
    return deco


def probe(V, d, R, seed=0):
    W = make_weight(V, d, seed, dev)
    h = (torch.randn(R, d, device=dev) * 1.2).to(torch.bfloat16)
    v = Verifier(d, V, max_batch=max(R, 1), gamma_max=1)
    rows = torch.arange(R, dtype=torch.int32, device=dev)
    outl = torch.full((R, V), float("nan"), device=dev)
    v.lmhead_logits(h, W, rows, outl)
    torch.cuda.synchronize()
    ref = h.float() @ W.float().t()
    err = (outl - ref).abs()
    return {"max_abs": float(err.max()), "mean_abs": float(err.mean()), "nan": int(torch.isnan(outl).sum()),
            "ref_std": float(ref.std())}


@stage("probe_small")
def _():
    return probe(1024, 128, 20)


@stage("probe_odd")
def _():
    return probe(1000, 64, 37)


@stage("probe_full")
def _():
    return probe(152064, 3584, 32)


def run_verify(b, path, V, d, B, dbg=True):
    v = Verifier(d, V, max_batch=B, gamma_max=int(b.gamma.max()) if b.gamma.max() > 0 else 1)
    v.set_option(NJ_OPT_PATH, path)
    acc = torch.empty(B, dtype=torch.int32, device=dev)
    nxt = torch.empty(B, dtype=torch.int32, device=dev)
    N, G = b.N, b.G
    d_ = {"lse": torch.full((N,), float("nan"), device=dev), "p_draft": torch.zeros(max(G, 1), device=dev),
          "mass": torch.zeros(B, dtype=torch.float64, device=dev), "flags": torch.zeros(B, dtype=torch.int32, device=dev)}
    v.verify(b.hidden, b.W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt, debug=d_ if dbg else None)
    torch.cuda.synchronize()
    return v, acc.cpu().numpy(), nxt.cpu().numpy(), {k: t.cpu().numpy() for k, t in d_.items()}


def compare(b, acc, nxt, dd):
    n = b.to_numpy()
    r = oracle.verify(n["hidden_bits"], n["W_bits"], n["draft_tokens"], n["draft_probs"], n["gamma"], n["uniforms"])
    tie = r["tie"]
    ok = (~tie)
    mis_acc = int(((acc != r["accept_len"]) & ok).sum())
    mis_tok = int(((nxt != r["next_token"]) & ok).sum())
    lse_err = float(np.nanmax(np.abs(dd["lse"] - r["lse"]))) if np.isfinite(dd["lse"]).any() else None
    pd_err = None
    if b.G:
        m = r["p_draft"] > 1e-30
        pd_err = float(np.max(np.abs(np.log(np.maximum(dd["p_draft"][:b.G][m], 1e-300)) - np.log(r["p_draft"][m]))))
    return {"B": b.B, "N": b.N, "mis_acc": mis_acc, "mis_tok": mis_tok, "ties": int(tie.sum()),
            "lse_maxerr": lse_err, "lnp_maxerr": pd_err, "flags": np.bincount(dd["flags"], minlength=8).tolist(),
            "acc_gpu": acc[:8].tolist(), "acc_or": r["accept_len"][:8].tolist(),
            "tok_gpu": nxt[:8].tolist(), "tok_or": r["next_token"][:8].tolist(),
            "mass_relerr": float(np.max(np.abs(dd["mass"] - r["mass"]) / np.maximum(r["mass"], 1e-300)))}


@stage("fused_toy")
def _():
    res = []
    for seed in range(6):
        b = make_batch(1, 3, V=32, d=16, seed=seed, device=dev)
        _, acc, nxt, dd = run_verify(b, NJ_PATH_FUSED, 32, 16, 1)
        res.append(compare(b, acc, nxt, dd))
    return {"runs": res}


@stage("twopass_toy")
def _():
    res = []
    for seed in range(6):
        b = make_batch(1, 3, V=32, d=16, seed=seed, device=dev)
        _, acc, nxt, dd = run_verify(b, NJ_PATH_TWOPASS, 32, 16, 1)
        res.append(compare(b, acc, nxt, dd))
    return {"runs": res}


@stage("fused_mid")
def _():
    b = make_batch(8, "mixed:5", V=8192, d=512, seed=3, device=dev)
    _, acc, nxt, dd = run_verify(b, NJ_PATH_FUSED, 8192, 512, 8)
    return compare(b, acc, nxt, dd)


@stage("twopass_mid")
def _():
    b = make_batch(40, "mixed:5", V=8192, d=512, seed=4, device=dev)
    _, acc, nxt, dd = run_verify(b, NJ_PATH_TWOPASS, 8192, 512, 40)
    return compare(b, acc, nxt, dd)


W_full = None


def get_wfull():
    global W_full
    if W_full is None:
        W_full = make_weight(152064, 3584, 0, dev)
    return W_full


@stage("fused_c2")
def _():
    get_wfull()
    b = make_batch(8, 3, V=152064, d=3584, seed=11, device=dev, W=W_full)
    v, acc, nxt, dd = run_verify(b, NJ_PATH_FUSED, 152064, 3584, 8)
    r = compare(b, acc, nxt, dd)
    # timing
    acc_t = torch.empty(8, dtype=torch.int32, device=dev)
    nxt_t = torch.empty(8, dtype=torch.int32, device=dev)
    for _ in range(3):
        v.verify(b.hidden, b.W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc_t, nxt_t)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        v.verify(b.hidden, b.W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc_t, nxt_t)
    e1.record()
    torch.cuda.synchronize()
    r["us_per_step"] = e0.elapsed_time(e1) / 20 * 1e3
    return r


@stage("twopass_c2")
def _():
    b = make_batch(8, 3, V=152064, d=3584, seed=11, device=dev, W=get_wfull())
    v, acc, nxt, dd = run_verify(b, NJ_PATH_TWOPASS, 152064, 3584, 8)
    r = compare(b, acc, nxt, dd)
    acc_t = torch.empty(8, dtype=torch.int32, device=dev)
    nxt_t = torch.empty(8, dtype=torch.int32, device=dev)
    for _ in range(3):
        v.verify(b.hidden, b.W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc_t, nxt_t)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        v.verify(b.hidden, b.W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc_t, nxt_t)
    e1.record()
    torch.cuda.synchronize()
    r["us_per_step"] = e0.elapsed_time(e1) / 20 * 1e3
    return r


@stage("twopass_big_timing")
def _():
    res = {}
    for B, g in [(64, 3), (256, 2), (256, 5)]:
        b = make_batch(B, g, V=152064, d=3584, seed=5, device=dev, W=get_wfull())
        v = Verifier(3584, 152064, max_batch=B, gamma_max=5)
        acc_t = torch.empty(B, dtype=torch.int32, device=dev)
        nxt_t = torch.empty(B, dtype=torch.int32, device=dev)
        for _ in range(3):
            v.verify(b.hidden, b.W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc_t, nxt_t)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            v.verify(b.hidden, b.W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc_t, nxt_t)
        e1.record()
        torch.cuda.synchronize()
        res[f"B{B}_g{g}_us"] = e0.elapsed_time(e1) / 10 * 1e3
        del v
    return res


json.dump(out, open("gpurun_out/gpu_check_%s.json" % ("_".join(SEL) or "all"), "w"), indent=1)
