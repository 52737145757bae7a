import ctypes, sys, json, torch
sys.path.insert(0, ".")
from paper_2512_22420_b200 import Verifier, load
from synth.inputs import make_weight
lib = load()
lib.nj_stream_test.argtypes = [ctypes.c_void_p]*3 + [ctypes.c_int32]*3 + [ctypes.c_void_p, ctypes.c_int32]
dev = torch.device("cuda:0")
V, d = 152064, 3584
W = make_weight(V, d, 0, dev)
H = torch.randn(64, d, device=dev).to(torch.bfloat16)
v = Verifier(d, V, max_batch=8, gamma_max=3)
for mode, group, S, hr in [(0,4,3,0),(0,4,2,0),(0,4,2,16),(0,4,2,32),(0,4,2,48),(0,2,4,32),(0,2,5,32),(0,3,3,32),(0,2,6,16),(0,8,1,0)]:
    st = torch.cuda.current_stream().cuda_stream
    rc = lib.nj_stream_test(v._h, st, W.data_ptr(), mode, group, S, H.data_ptr() if hr else None, hr)
    if rc: print("rc", rc, mode, group, S, hr); continue
    for _ in range(2): lib.nj_stream_test(v._h, st, W.data_ptr(), mode, group, S, H.data_ptr() if hr else None, hr)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): lib.nj_stream_test(v._h, st, W.data_ptr(), mode, group, S, H.data_ptr() if hr else None, hr)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    print(f"G={group} S={S} hrows={hr}: {us:.1f} us  W-TB/s {V*d*2/us/1e6:.3f}", flush=True)
