"""tcgen05.mma issue rate: cycles per 4-MMA group (M=128, N=n, K=16 each)."""
import ctypes, sys, torch
sys.path.insert(0, ".")
from scripts.probes import _probe
dev = torch.device("cuda:0")
out = torch.zeros(148, dtype=torch.int64, device=dev)
for mode in (0, 2, 1):
    for n in (32, 64, 128, 256):
        for _ in range(2):
            _probe.mma_probe(n, 4096, mode, out)
        torch.cuda.synchronize()
        c = out.float()
        ideal = 4 * 128 * n / 256
        print(f"mode {mode} N={n}: cycles/group median {c.median():.0f} (min {c.min():.0f} max {c.max():.0f}); tensor floor {ideal:.0f}", flush=True)
