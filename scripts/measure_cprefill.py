"""B200 analogue of PAPER Table 1: the
switching cost c_prefill(L_max, B) of re-enabling speculation, i.e. the draft
model's KV-cache reconstruction -- a forward pass over the L_max tokens each of
the B requests generated while speculation was off, attending to its existing
context -- measured on this GPU for a synthetic 0.5B-shaped draft (Qwen2-0.5B
geometry: 24 layers, d = 896, 14 query / 2 KV heads of 64, SwiGLU FFN 4864,
vocabulary 151936; random bf16 weights, no checkpoint exists here).

This is a MEASUREMENT feeding the host bandit's lookup table (nj_bandit_create
cost_ms), not part of the verification hot path: it uses plain torch ops
(cuBLAS GEMMs, SDPA attention with GQA reading the KV cache in place) under a
CUDA graph, median of 20 replays.

    python scripts/measure_cprefill.py [--ctx 1024] [--out profiles/r02_cprefill_b200.csv]

Writes the CSV (input_len, batch_size, cost_ms; the format of
tests/golden/table1_cprefill.csv) and a JSON with the full grid beside it.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LAYERS, D, HQ, HKV, HD, FF, VOCAB = 24, 896, 14, 2, 64, 4864, 151936


def make_weights(dev, seed=0):
    g = torch.Generator(device=dev).manual_seed(seed)
    r = lambda *s: (torch.randn(*s, device=dev, generator=g) * 0.02).to(torch.bfloat16)
    layers = []
    for _ in range(LAYERS):
        layers.append({"wqkv": r(D, (HQ + 2 * HKV) * HD), "wo": r(HQ * HD, D), "wgu": r(D, 2 * FF), "wd": r(FF, D),
                       "n1": torch.ones(D, device=dev, dtype=torch.bfloat16),
                       "n2": torch.ones(D, device=dev, dtype=torch.bfloat16)})
    return layers, r(D, VOCAB)


def rms(x, w):
    return (x.float() * torch.rsqrt(x.float().pow(2).mean(-1, keepdim=True) + 1e-6)).to(x.dtype) * w


def prefill(x, kcache, vcache, layers, lm, mask, ctx):
    """x [B, L, D] new tokens; kcache/vcache per layer [B, HKV, ctx + L, HD] (the
    first ctx positions already filled); the new keys / values are written in
    place and attention reads the cache directly (GQA, no KV copies); returns
    the last position's logits (the draft then proposes from it)."""
    B, L, _ = x.shape
    for li, p in enumerate(layers):
        h = rms(x, p["n1"])
        qkv = h @ p["wqkv"]
        q, k, v = qkv.split([HQ * HD, HKV * HD, HKV * HD], dim=-1)
        q = q.view(B, L, HQ, HD).transpose(1, 2)
        kcache[li][:, :, ctx:] = k.view(B, L, HKV, HD).transpose(1, 2)
        vcache[li][:, :, ctx:] = v.view(B, L, HKV, HD).transpose(1, 2)
        a = torch.nn.functional.scaled_dot_product_attention(q, kcache[li], vcache[li], attn_mask=mask,
                                                             enable_gqa=True)
        x = x + a.transpose(1, 2).reshape(B, L, HQ * HD) @ p["wo"]
        h = rms(x, p["n2"])
        gu = h @ p["wgu"]
        gt, up = gu.chunk(2, dim=-1)
        x = x + (torch.nn.functional.silu(gt) * up) @ p["wd"]
    return x[:, -1] @ lm


def measure(L, B, ctx, layers, lm, dev, reps=20):
    x = (torch.randn(B, L, D, device=dev) * 0.5).to(torch.bfloat16)
    kc = [(torch.randn(B, HKV, ctx + L, HD, device=dev) * 0.5).to(torch.bfloat16) for _ in range(LAYERS)]
    vc = [(torch.randn(B, HKV, ctx + L, HD, device=dev) * 0.5).to(torch.bfloat16) for _ in range(LAYERS)]
    # causal over the new tokens, full over the cached context (bottom-right aligned);
    # one new token attends to everything (no mask)
    mask = None if L == 1 else torch.ones(L, ctx + L, dtype=torch.bool, device=dev).tril(diagonal=ctx)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            prefill(x, kc, vc, layers, lm, mask, ctx)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            prefill(x, kc, vc, layers, lm, mask, ctx)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        g.replay()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    del g, kc, vc, x
    torch.cuda.empty_cache()
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, default=1024, help="tokens already in the draft's KV cache per request")
    ap.add_argument("--lens", default="1,2,4,8,16,32,64,128,256,512")
    ap.add_argument("--batches", default="1,8,16,32,64,128,256")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_cprefill_b200.csv"))
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    layers, lm = make_weights(dev)
    Ls = [int(x) for x in a.lens.split(",")]
    Bs = [int(x) for x in a.batches.split(",")]
    grid = {}
    for L in Ls:
        for B in Bs:
            ms = measure(L, B, a.ctx, layers, lm, dev)
            grid[f"{L},{B}"] = ms
            print(f"L={L:4d} B={B:4d}: {ms:8.3f} ms", flush=True)
    with open(a.out, "w") as f:
        f.write(f"# B200-measured c_prefill (ms): synthetic 0.5B-shaped draft KV reconstruction of L new tokens\n"
                f"# per request over a {a.ctx}-token cached context, B requests (scripts/measure_cprefill.py)\n")
        f.write("input_len,batch_size,cost_ms\n")
        for L in Ls:
            for B in Bs:
                f.write(f"{L},{B},{grid[f'{L},{B}']:.4f}\n")
    json.dump({"device": torch.cuda.get_device_name(0), "ctx": a.ctx,
               "model": {"layers": LAYERS, "d": D, "heads_q": HQ, "heads_kv": HKV, "head_dim": HD, "ffn": FF,
                         "vocab": VOCAB},
               "how": "torch bf16 (cuBLAS GEMMs, SDPA), one CUDA graph per (L, B), median of 20 replays",
               "grid_ms": grid}, open(os.path.splitext(a.out)[0] + ".json", "w"), indent=1)
    print(a.out)


if __name__ == "__main__":
    sys.exit(main())
