"""cuBLAS (torch.matmul, bf16 in / bf16 out) on the LM-head shape: the library's rate on the same GEMM."""
import torch

dev = torch.device("cuda:0")
V, d = 152064, 3584
W = (torch.randn(V, d, device=dev) * 0.05).to(torch.bfloat16)
for R in (128, 256, 512, 1024, 1536):
    h = torch.randn(R, d, device=dev).to(torch.bfloat16)
    for _ in range(3):
        out = h @ W.t()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = h @ W.t()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    t = sorted(ts)[5]
    print(f"cuBLAS R={R:5d} {t:8.1f} us {2 * R * V * d / t / 1e6:7.1f} TF/s", flush=True)
