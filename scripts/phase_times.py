import ctypes, sys, json, numpy as np, torch
sys.path.insert(0, ".")
from paper_2512_22420_b200 import NJ_OPT_PATH, NJ_PATH_FUSED, NJ_OPT_CERTIFY, Verifier, load
from synth.inputs import make_batch, make_weight
lib = load(); lib.nj_debug_phase_times.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
dev = torch.device("cuda:0"); V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
for B, g in [(8, 3), (1, 0), (16, 2)]:
    b = make_batch(B, g, V=V, d=d, seed=0, device=dev, W=W)
    v = Verifier(d, V, max_batch=B, gamma_max=5); v.set_option(NJ_OPT_PATH, NJ_PATH_FUSED); v.set_option(NJ_OPT_CERTIFY, 0)
    acc = torch.empty(B, dtype=torch.int32, device=dev); nxt = torch.empty(B, dtype=torch.int32, device=dev)
    for _ in range(5): v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
    torch.cuda.synchronize()
    ts = np.zeros(16 * 1024, np.uint64)
    lib.nj_debug_phase_times(v._h, ts.ctypes.data, 16 * 1024)
    grid = 132
    t = ts[:grid * 16].reshape(grid, 16).astype(np.int64)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    names = ["start", "p1_done", "bar1", "lsel", "lse", "accept", "qready", "weights", "mass", "bar2", "-", "prefix", "end"]
    med = [float(np.median(rel[:, i])) for i in range(len(names))]
    mx = [float(rel[:, i].max()) for i in range(len(names))]
    print(f"B={B} g={g}: " + " ".join(f"{n}={med[i]:.1f}/{mx[i]:.1f}" for i, n in enumerate(names) if n != "-"), flush=True)
