import ctypes, os, sys, torch
sys.path.insert(0, ".")
from paper_2512_22420_b200 import Verifier, load
from synth.inputs import make_weight
lib = load()
dev = torch.device("cuda:0"); V, d = 152064, 3584
W = make_weight(V, d, 0, dev); H = torch.randn(64, d, device=dev).to(torch.bfloat16)
v = Verifier(d, V, max_batch=8, gamma_max=3)
for G, S, hr in [(4, 3, 0), (4, 2, 32), (4, 2, 0)]:
    st = torch.cuda.current_stream().cuda_stream
    args = (v._h, st, W.data_ptr(), 0, G, S, H.data_ptr() if hr else None, hr)
    for _ in range(2): lib.nj_stream_test(*args)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): lib.nj_stream_test(*args)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    print(f"grid={os.environ.get('NJ_GRID','148')} G={G} S={S} hrows={hr}: {us:.1f} us  {V*d*2/us/1e6:.3f} TB/s", flush=True)
