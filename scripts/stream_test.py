import ctypes, sys, json, torch
sys.path.insert(0, ".")
from scripts.probes import _probe
from synth.inputs import make_weight
dev = torch.device("cuda:0")
V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
nkb = d // 64
Wp = W.view(V // 128, 128, nkb, 64).permute(0, 2, 1, 3).contiguous()   # [tile][kb][128][64]
res = {}
for mode, group, S, Wt in [(0,1,12,W),(0,1,8,W),(1,2,6,W),(1,4,3,W),(2,1,12,Wp),(2,1,8,Wp),(2,2,6,Wp),(2,4,3,Wp)]:
    for _ in range(3): _probe.stream_test(Wt, mode, group, S, V=V, d=d)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): _probe.stream_test(Wt, mode, group, S, V=V, d=d)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    res[f"mode{mode}_g{group}_S{S}"] = {"us": round(us, 1), "TBps": round(V * d * 2 / us / 1e6, 3)}
    print(mode, group, S, res[f"mode{mode}_g{group}_S{S}"], flush=True)
# reference: torch copy of W
out = torch.empty_like(W)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): out.copy_(W)
e1.record(); torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 10 * 1e3
print("torch copy (r+w)", round(us, 1), "us", round(2 * V * d * 2 / us / 1e6, 3), "TB/s")
