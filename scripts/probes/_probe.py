"""libnj_probe.so: measurement probes outside the product library (see
nj_probe.cu).  build() compiles it for sm_100a; the functions take torch
tensors and launch on the current stream."""
from __future__ import annotations

import ctypes
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
CSRC = os.path.join(ROOT, "paper_2512_22420_b200", "csrc")
LIB = os.path.join(HERE, "libnj_probe.so")
SRC = ["nj_probe.cu", "nj_probe_ks.cuh", "nj_stream_test.cuh", "nj_mma_probe.cuh", "nj_tmem_bw.cuh"]
_lib = None


def build(force: bool = False) -> str:
    deps = [os.path.join(HERE, f) for f in SRC] + [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    if not force and os.path.exists(LIB) and all(os.path.getmtime(p) <= os.path.getmtime(LIB) for p in deps):
        return LIB
    tmp = LIB + ".tmp.%d" % os.getpid()
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                           "-Xcompiler", "-fPIC", "-shared", "-I", CSRC, "-I", HERE, "--expt-relaxed-constexpr",
                           "-diag-suppress", "177", "-o", tmp, os.path.join(HERE, "nj_probe.cu")])
    os.replace(tmp, LIB)
    return LIB


def load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        lib.njp_logits_ks.argtypes = [P, P, I32, I32, P, I32, P, I64, I32]
        lib.njp_stream_test.argtypes = [P, P, I32, I32, I32, I32, I32, P, I32, I32]
        lib.njp_mma_probe.argtypes = [P, I32, I32, I32, P]
        lib.njp_mma_probe_cg2.argtypes = [P, I32, I32, I32, P]
        lib.njp_tmem_bw.argtypes = [P, I32, I32, I32, I32, I32, P]
        for f in (lib.njp_logits_ks, lib.njp_stream_test, lib.njp_mma_probe, lib.njp_mma_probe_cg2, lib.njp_tmem_bw):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _st():
    import torch
    return torch.cuda.current_stream().cuda_stream


def _ok(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed ({rc})")


def logits_ks(hidden, W, out64, ks: int):
    """out64[r] = fp64 sum of ks-MMA fresh-accumulator partials of W @ hidden[r]."""
    V, d = W.shape
    _ok(load().njp_logits_ks(_st(), W.data_ptr(), V, d, hidden.data_ptr(), hidden.shape[0], out64.data_ptr(),
                             out64.stride(0), ks), "njp_logits_ks")


def stream_test(W, mode: int, group: int, nstages: int, H=None, hrows: int = 0, grid: int = 0, V=None, d=None):
    V = V or W.shape[0]
    d = d or W.shape[-1]
    _ok(load().njp_stream_test(_st(), W.data_ptr(), V, d, mode, group, nstages,
                               H.data_ptr() if H is not None else None, hrows, grid), "njp_stream_test")


def mma_probe(n: int, iters: int, mode: int, out):
    _ok(load().njp_mma_probe(_st(), n, iters, mode, out.data_ptr()), "njp_mma_probe")


def mma_probe_cg2(n: int, iters: int, mode: int, out):
    _ok(load().njp_mma_probe_cg2(_st(), n, iters, mode, out.data_ptr()), "njp_mma_probe_cg2")


def tmem_bw(nwarps: int, x: int, inflight: int, cols: int, rounds: int, out):
    """TMEM read probe: out [2 * SMs] int64 (cycles, checksum) per CTA."""
    _ok(load().njp_tmem_bw(_st(), nwarps, x, inflight, cols, rounds, out.data_ptr()), "njp_tmem_bw")
