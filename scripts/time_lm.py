"""Time the production LM-head GEMM (nj_lmhead_logits -> k_lmhead, WRITE|STATS) at the Qwen shape.

usage: python scripts/time_lm.py R[,R...] [ENV=V ...]   (each env combo spec 'A=1;B=2' as extra args)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_22420_b200 import Verifier  # noqa: E402

V, d = 152064, 3584
dev = torch.device("cuda:0")
Rs = [int(x) for x in sys.argv[1].split(",")]
combos = sys.argv[2:] or [""]
try:
    import pynvml as nv
    nv.nvmlInit()
    nvh = nv.nvmlDeviceGetHandleByIndex(0)
except Exception:   # noqa: BLE001
    nv = None
g = torch.Generator(device=dev).manual_seed(0)
W = (torch.randn(V, d, device=dev, generator=g) * 0.05).to(torch.bfloat16)
Rmax = max(Rs)
h = torch.randn(Rmax, d, device=dev, generator=g).to(torch.bfloat16)
out = torch.empty(Rmax, V, device=dev)
for combo in combos:
    env = dict(kv.split("=") for kv in combo.split(";") if kv)
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    for R in Rs:
        mb = min(R, 768)
        v = Verifier(d, V, max_batch=mb, gamma_max=(R + mb - 1) // mb)
        rows = torch.arange(R, dtype=torch.int32, device=dev)
        for _ in range(3):
            v.lmhead_logits(h, W, rows, out)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            v.lmhead_logits(h, W, rows, out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        t = ts[len(ts) // 2]
        # SM clock while the kernel runs back to back (nvml, ~every 2 ms)
        clk = []
        if nv is not None:
            import threading
            stop = threading.Event()

            def samp():
                while not stop.is_set():
                    clk.append(nv.nvmlDeviceGetClockInfo(nvh, nv.NVML_CLOCK_SM))
                    stop.wait(0.002)
            th = threading.Thread(target=samp)
            th.start()
            for _ in range(int(max(20, 60000 / max(t, 1)))):
                v.lmhead_logits(h, W, rows, out)
            torch.cuda.synchronize()
            stop.set()
            th.join()
        mhz = sorted(clk)[len(clk) // 2] if clk else 0
        fl = 2.0 * R * V * d
        hbm = (2.0 * V * d + 4.0 * R * V) / 6541.8e9 * 1e6
        print(f"{combo or 'default':28s} R={R:5d} {t:8.1f} us  {fl / t / 1e6:7.1f} TF/s  "
              f"(t*={max(fl / 1646.9e12 * 1e6, hbm):.0f} us, frac {max(fl / 1646.9e12 * 1e6, hbm) / t:.2f})  "
              f"sm {mhz} MHz = {t * mhz:.3g} cycles", flush=True)
        v.close()
    for k, val in saved.items():
        if val is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = val
