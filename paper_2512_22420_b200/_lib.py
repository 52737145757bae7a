"""Thin ctypes binding of libnj (include/nj.h).  Argument marshalling only.

Every step of the verification path runs in libnj's CUDA kernels; this module
only converts torch tensors / numpy arrays to raw pointers.  There is no CPU
fallback: if libnj.so is missing or no sm_100 device is visible, calls raise.

Names follow the C ABI: nj_create, nj_verify, nj_verify_host, nj_plan,
nj_set_option, nj_lmhead_logits, nj_sample_from_logits, nj_select_gamma,
nj_observe, nj_bandit_* ...  `Verifier` and `Bandit` are small RAII wrappers.
"""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libnj.so")

NJ_OK, NJ_EINVAL, NJ_ESHAPE, NJ_ECUDA, NJ_ENCCL, NJ_ENOMEM, NJ_EUNSUPPORTED = range(7)
NJ_PATH_AUTO, NJ_PATH_FUSED, NJ_PATH_TWOPASS, NJ_PATH_STAGED = 0, 1, 2, 3
NJ_OPT_PATH, NJ_OPT_CERTIFY, NJ_OPT_FORCE_FALLBACK, NJ_OPT_PROFILE, NJ_OPT_Q_ZERO_COPY, NJ_OPT_Q_STAGE_ROWS = 1, 2, 3, 4, 5, 6
NJ_FLAG_FALLBACK, NJ_FLAG_ZERO_MASS, NJ_FLAG_CLAMP = 1, 2, 4

# every symbol include/nj.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "nj_create", "nj_destroy", "nj_last_error", "nj_verify", "nj_verify_host", "nj_set_option", "nj_set_temperature",
    "nj_plan",
    "nj_kernel_time",
    "nj_lmhead_logits", "nj_sample_from_logits", "nj_bandit_create", "nj_bandit_destroy", "nj_select_gamma",
    "nj_observe", "nj_exploitation_score", "nj_prefill_cost_ms", "nj_bandit_state", "nj_bandit_arm",
    "nj_bandit_last_gamma", "nj_bandit_snapshot_json",
    "nj_shard_range", "nj_nccl_get_unique_id", "nj_nccl_comm_init", "nj_nccl_comm_destroy", "nj_group_create",
    "nj_group_destroy", "nj_group_member", "nj_group_last_error", "nj_group_verify",
    "nj_propose", "nj_verify_greedy", "nj_host_staged_rows",
]
NJ_NCCL_ID_BYTES = 128


class NJError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"libnj status {status}: {msg}")
        self.status = status


class NJArgError(NJError, ValueError):
    """Argument rejected by the binding's checks before any pointer crosses the
    C ABI (the same status codes the library uses: NJ_EINVAL / NJ_ESHAPE)."""

    def __init__(self, status, msg):
        super().__init__(status, msg)


class nj_config(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int32), ("V", ctypes.c_int32), ("max_batch", ctypes.c_int32),
                ("gamma_max", ctypes.c_int32), ("device", ctypes.c_int32), ("nccl_comm", ctypes.c_void_p),
                ("v_begin", ctypes.c_int32), ("v_end", ctypes.c_int32)]


class nj_debug(ctypes.Structure):
    _fields_ = [("lse", ctypes.c_void_p), ("p_draft", ctypes.c_void_p), ("mass", ctypes.c_void_p),
                ("flags", ctypes.c_void_p)]


_lib = None


def load():
    """Load libnj.so (never builds, never falls back)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not found: run `python -m paper_2512_22420_b200._build` "
                          "(libnj has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I32, I64, U64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
    sig = {
        "nj_create": ([ctypes.POINTER(nj_config), ctypes.POINTER(P)], I32),
        "nj_destroy": ([P], None),
        "nj_last_error": ([P], ctypes.c_char_p),
        "nj_verify": ([P, P, P, P, P, P, I64, P, P, I32, P, P, P], I32),
        "nj_verify_host": ([P, P, P, P, P, P, I64, P, P, I32, P, P], I32),
        "nj_host_staged_rows": ([P, P, I32, P], I32),
        "nj_set_option": ([P, I32, I64], I32),
        "nj_set_temperature": ([P, D], I32),
        "nj_plan": ([P, P, I32, P, P], I32),
        "nj_kernel_time": ([P, P, P, I32], I32),
        "nj_lmhead_logits": ([P, P, P, P, P, I32, P, I64, I32], I32),
        "nj_sample_from_logits": ([P, P, P, I64, P, P, I64, P, I32, P, P], I32),
        "nj_propose": ([P, P, P, P, P, I32, P, P, I64], I32),
        "nj_verify_greedy": ([P, P, P, P, P, P, I32, P, P], I32),
        "nj_bandit_create": ([I32, I32, U64, P, I32, P, I32, P, ctypes.POINTER(P)], I32),
        "nj_bandit_destroy": ([P], None),
        "nj_select_gamma": ([P, I32, I32], I32),
        "nj_observe": ([P, I32, I32, D], I32),
        "nj_exploitation_score": ([P, I32, I32, I32, I32], D),
        "nj_prefill_cost_ms": ([P, I32, I32], D),
        "nj_bandit_state": ([P, I32, P, P, P, P, P], I32),
        "nj_bandit_arm": ([P, I32, I32, P, P], I32),
        "nj_bandit_last_gamma": ([P], I32),
        "nj_bandit_snapshot_json": ([P, P, ctypes.c_size_t, P], I32),
        "nj_shard_range": ([I32, I32, I32, P, P], I32),
        "nj_nccl_get_unique_id": ([P], I32),
        "nj_nccl_comm_init": ([I32, P, I32, I32, ctypes.POINTER(P)], I32),
        "nj_nccl_comm_destroy": ([P], None),
        "nj_group_create": ([ctypes.POINTER(nj_config), I32, ctypes.POINTER(P)], I32),
        "nj_group_destroy": ([P], None),
        "nj_group_member": ([P, I32], P),
        "nj_group_last_error": ([P], ctypes.c_char_p),
        "nj_group_verify": ([P, P, P, P, P, P, I64, P, P, I32, P, P, P], I32),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def _ptr(t):
    """Raw pointer of a torch tensor / numpy array / None."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _dev(t, name: str, dtype: str, rowmajor: bool = False, host: bool = False, min_rows: int = 0,
         min_numel: int = 0, ncols: int | None = None, min_cols: int | None = None):
    """Argument check before a raw pointer crosses the C ABI: a torch tensor on
    the right kind of device with the dtype the ABI expects, and a layout the
    kernels can index (contiguous; or, with rowmajor, 2-D with unit column
    stride and any row pitch).  Raises NJArgError (an NJError and a ValueError)
    instead of letting the library misread memory."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise NJArgError(NJ_EINVAL, f"{name}: expected a torch.Tensor, got {type(t).__name__}")
    if t.dtype != getattr(torch, dtype):
        raise NJArgError(NJ_EINVAL, f"{name}: dtype {t.dtype}, expected torch.{dtype}")
    if host and t.is_cuda:
        raise NJArgError(NJ_EINVAL, f"{name}: expected a host (CPU) tensor")
    if not host and not t.is_cuda:
        raise NJArgError(NJ_EINVAL, f"{name}: expected a CUDA tensor")
    if rowmajor:
        if t.dim() != 2 or (t.shape[1] > 1 and t.stride(1) != 1) or t.stride(0) < t.shape[1]:
            raise NJArgError(NJ_ESHAPE, f"{name}: expected a 2-D row-major tensor (unit column stride), "
                             f"shape {tuple(t.shape)} strides {t.stride()}")
    elif not t.is_contiguous():
        raise NJArgError(NJ_ESHAPE, f"{name}: expected a contiguous tensor, strides {t.stride()}")
    if min_rows and (t.dim() < 1 or t.shape[0] < min_rows):
        raise NJArgError(NJ_ESHAPE, f"{name}: needs >= {min_rows} rows, shape {tuple(t.shape)}")
    if min_numel and t.numel() < min_numel:
        raise NJArgError(NJ_ESHAPE, f"{name}: needs >= {min_numel} elements, has {t.numel()}")
    if ncols is not None and (t.dim() != 2 or t.shape[1] != ncols):
        raise NJArgError(NJ_ESHAPE, f"{name}: expected {ncols} columns, shape {tuple(t.shape)}")
    if min_cols is not None and (t.dim() != 2 or t.shape[1] < min_cols):
        raise NJArgError(NJ_ESHAPE, f"{name}: expected >= {min_cols} columns, shape {tuple(t.shape)}")
    return t


def _check_batch(cfg, hidden, W, draft_tokens, draft_probs, g, uniforms, accept_len, next_token, host=False,
                 ldq=None):
    """Shape / dtype / layout checks of one nj_verify-style call (include/nj.h)."""
    B, G = int(g.shape[0]), int(g.sum())
    N = G + B
    _dev(hidden, "hidden", "bfloat16", host=host, min_rows=N, ncols=cfg.d)
    if W is not None:
        _dev(W, "W_lm", "bfloat16", ncols=cfg.d, min_rows=cfg.v_end - cfg.v_begin)
    _dev(uniforms, "uniforms", "float32", host=host, min_numel=N)
    _dev(accept_len, "accept_len", "int32", host=host, min_numel=B)
    _dev(next_token, "next_token", "int32", host=host, min_numel=B)
    if G > 0:
        _dev(draft_tokens, "draft_tokens", "int32", host=host, min_numel=G)
        _dev(draft_probs, "draft_probs", "float32", rowmajor=ldq is None, host=host, min_rows=G,
             min_cols=cfg.V if ldq is None else None)


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


class Verifier:
    """RAII wrapper of nj_ctx (unsharded unless v_begin/v_end/nccl_comm given)."""

    def __init__(self, d: int, V: int, max_batch: int, gamma_max: int, device: int = 0,
                 v_begin: int = 0, v_end: int | None = None, nccl_comm=None):
        lib = load()
        cfg = nj_config(d, V, max_batch, gamma_max, device, nccl_comm, v_begin, V if v_end is None else v_end)
        h = ctypes.c_void_p()
        st = lib.nj_create(ctypes.byref(cfg), ctypes.byref(h))
        if st != NJ_OK:
            raise NJError(st, lib.nj_last_error(None).decode())
        self._lib, self._h, self.cfg = lib, h, cfg

    def close(self):
        if self._h:
            self._lib.nj_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st != NJ_OK:
            raise NJError(st, self._lib.nj_last_error(self._h).decode())

    def set_option(self, opt: int, value: int):
        self._check(self._lib.nj_set_option(self._h, opt, int(value)))

    def set_temperature(self, temperature: float):
        """nj_set_temperature: target distribution softmax(l / T) for later calls."""
        self._check(self._lib.nj_set_temperature(self._h, float(temperature)))

    def plan(self, gamma):
        g = np.ascontiguousarray(gamma, np.int32)
        path, n = ctypes.c_int32(), ctypes.c_int32()
        self._check(self._lib.nj_plan(self._h, _ptr(g), g.shape[0], ctypes.byref(path), ctypes.byref(n)))
        return path.value, n.value

    def kernel_time(self, reset: bool = True):
        """(ms_total, launches) of the dominant kernel since the last reset (NJ_OPT_PROFILE)."""
        ms, n = ctypes.c_double(), ctypes.c_int64()
        self._check(self._lib.nj_kernel_time(self._h, ctypes.byref(ms), ctypes.byref(n), int(reset)))
        return ms.value, n.value

    def verify(self, hidden, W, draft_tokens, draft_probs, gamma, uniforms, accept_len, next_token,
               debug: dict | None = None, stream=None):
        """nj_verify on device tensors; outputs written into accept_len / next_token."""
        g = np.ascontiguousarray(gamma, np.int32)
        _check_batch(self.cfg, hidden, W, draft_tokens, draft_probs, g, uniforms, accept_len, next_token)
        dbg = None
        if debug is not None:
            B, N, G = int(g.shape[0]), int(g.sum()) + int(g.shape[0]), int(g.sum())
            for k, dt, n in (("lse", "float32", N), ("p_draft", "float32", G), ("mass", "float64", B),
                             ("flags", "int32", B)):
                if debug.get(k) is not None:
                    _dev(debug[k], "debug." + k, dt, min_numel=n)
            dbg = nj_debug(_ptr(debug.get("lse")), _ptr(debug.get("p_draft")), _ptr(debug.get("mass")),
                           _ptr(debug.get("flags")))
        self._check(self._lib.nj_verify(
            self._h, _stream(stream), _ptr(hidden), _ptr(W), _ptr(draft_tokens), _ptr(draft_probs),
            int(draft_probs.stride(0)) if draft_probs is not None else int(self.cfg.V), _ptr(g), _ptr(uniforms),
            g.shape[0], _ptr(accept_len), _ptr(next_token), ctypes.byref(dbg) if dbg is not None else None))

    def verify_host(self, hidden_h, W, tok_h, q_h, gamma, u_h, acc_h, next_h, ldq=None, stream=None):
        """nj_verify_host: host (pinned) inputs/outputs, resident W; synchronous."""
        g = np.ascontiguousarray(gamma, np.int32)
        _check_batch(self.cfg, hidden_h, W, tok_h, q_h, g, u_h, acc_h, next_h, host=True, ldq=ldq)
        ldq = int(q_h.stride(0)) if ldq is None else ldq
        self._check(self._lib.nj_verify_host(
            self._h, _stream(stream), _ptr(hidden_h), _ptr(W), _ptr(tok_h), _ptr(q_h), ldq, _ptr(g),
            _ptr(u_h), g.shape[0], _ptr(acc_h), _ptr(next_h)))

    def host_staged_rows(self):
        """nj_host_staged_rows: the draft rows the last verify_host staged to the device."""
        n = ctypes.c_int32(0)
        self._check(self._lib.nj_host_staged_rows(self._h, None, 0, ctypes.byref(n)))
        rows = np.zeros(max(n.value, 1), np.int32)
        self._check(self._lib.nj_host_staged_rows(self._h, rows.ctypes.data, n.value, ctypes.byref(n)))
        return rows[:n.value]

    def lmhead_logits(self, hidden, W, rows, out, ks: int = 0, stream=None):
        """nj_lmhead_logits: fp32 logits of hidden[rows] through the production GEMM."""
        _dev(hidden, "hidden", "bfloat16")
        _dev(W, "W", "bfloat16")
        _dev(rows, "rows", "int32")
        _dev(out, "out", "float32", rowmajor=True)
        self._check(self._lib.nj_lmhead_logits(self._h, _stream(stream), _ptr(hidden), _ptr(W), _ptr(rows),
                                               int(rows.shape[0]), _ptr(out), int(out.stride(0)), int(ks)))

    def verify_greedy(self, hidden, W, draft_tokens, gamma, accept_len, next_token, stream=None):
        """nj_verify_greedy: verification against the argmax target (include/nj.h)."""
        g = np.ascontiguousarray(np.asarray(gamma, dtype=np.int32))
        B, G = int(g.shape[0]), int(g.sum())
        _dev(hidden, "hidden", "bfloat16", min_rows=G + B, ncols=self.cfg.d)
        _dev(W, "W_lm", "bfloat16", ncols=self.cfg.d)
        _dev(accept_len, "accept_len", "int32", min_numel=B)
        _dev(next_token, "next_token", "int32", min_numel=B)
        if G:
            _dev(draft_tokens, "draft_tokens", "int32", min_numel=G)
        self._check(self._lib.nj_verify_greedy(
            self._h, _stream(stream), _ptr(hidden), _ptr(W), _ptr(draft_tokens), g.ctypes.data, g.shape[0],
            _ptr(accept_len), _ptr(next_token)))

    def propose(self, hidden, W, u, tokens, q_out, stream=None):
        """nj_propose: draft LM head + softmax + inverse-CDF draw (include/nj.h):
        tokens[b] ~ q_out[b] = softmax(W @ hidden[b]) with uniform u[b]."""
        B = int(hidden.shape[0])
        _dev(hidden, "hidden", "bfloat16", ncols=self.cfg.d)
        _dev(W, "W_lm", "bfloat16", ncols=self.cfg.d)
        _dev(u, "u", "float32", min_numel=B)
        _dev(tokens, "tokens", "int32", min_numel=B)
        _dev(q_out, "q_out", "float32", rowmajor=True, min_rows=B, min_cols=self.cfg.V)
        self._check(self._lib.nj_propose(
            self._h, _stream(stream), _ptr(hidden), _ptr(W), _ptr(u), int(hidden.shape[0]), _ptr(tokens),
            _ptr(q_out), int(q_out.stride(0))))

    def sample_from_logits(self, logits, residual, q, u, next_token, mass=None, stream=None):
        B = int(logits.shape[0])
        _dev(logits, "logits", "float32", rowmajor=True, min_cols=self.cfg.V)
        _dev(residual, "residual", "int32", min_numel=B)
        _dev(q, "q", "float32", rowmajor=True, min_rows=B, min_cols=self.cfg.V)
        _dev(u, "u", "float32", min_numel=B)
        _dev(next_token, "next_token", "int32", min_numel=B)
        if mass is not None:
            _dev(mass, "mass", "float64", min_numel=B)
        self._check(self._lib.nj_sample_from_logits(
            self._h, _stream(stream), _ptr(logits), int(logits.stride(0)), _ptr(residual), _ptr(q),
            int(q.stride(0)), _ptr(u), int(logits.shape[0]), _ptr(next_token), _ptr(mass)))


def shard_range(V: int, nranks: int, rank: int):
    """nj_shard_range: [v_begin, v_end) of `rank` (128-row aligned, rank order)."""
    lib = load()
    vb, ve = ctypes.c_int32(), ctypes.c_int32()
    st = lib.nj_shard_range(V, nranks, rank, ctypes.byref(vb), ctypes.byref(ve))
    if st != NJ_OK:
        raise NJError(st, f"nj_shard_range({V}, {nranks}, {rank})")
    return vb.value, ve.value


def nccl_unique_id() -> bytes:
    """nj_nccl_get_unique_id (rank 0); broadcast the bytes to the other ranks."""
    buf = ctypes.create_string_buffer(NJ_NCCL_ID_BYTES)
    st = load().nj_nccl_get_unique_id(buf)
    if st != NJ_OK:
        raise NJError(st, "nj_nccl_get_unique_id")
    return buf.raw


class NcclComm:
    """RAII wrapper of the communicator libnj creates (nj_nccl_comm_init)."""

    def __init__(self, nranks: int, uid: bytes, rank: int, device: int):
        lib = load()
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(bytes(uid), NJ_NCCL_ID_BYTES)
        st = lib.nj_nccl_comm_init(nranks, buf, rank, device, ctypes.byref(h))
        if st != NJ_OK:
            raise NJError(st, f"nj_nccl_comm_init(rank {rank} of {nranks})")
        self._lib, self.handle, self.nranks, self.rank = lib, h.value, nranks, rank

    def close(self):
        if self.handle:
            self._lib.nj_nccl_comm_destroy(self.handle)
            self.handle = None


class ShardGroup:
    """RAII wrapper of nj_group: `nshards` vocab shards on one device, exchanges
    as device copies (the per-rank kernels of the NCCL mode, in one process)."""

    def __init__(self, d: int, V: int, max_batch: int, gamma_max: int, nshards: int, device: int = 0):
        lib = load()
        cfg = nj_config(d, V, max_batch, gamma_max, device, None, 0, V)
        h = ctypes.c_void_p()
        st = lib.nj_group_create(ctypes.byref(cfg), nshards, ctypes.byref(h))
        if st != NJ_OK:
            raise NJError(st, lib.nj_group_last_error(None).decode())
        self._lib, self._h, self.n, self.cfg = lib, h, nshards, cfg
        self.ranges = [shard_range(V, nshards, r) for r in range(nshards)]

    def close(self):
        if self._h:
            self._lib.nj_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, opt: int, value: int):
        for r in range(self.n):
            m = self._lib.nj_group_member(self._h, r)
            st = self._lib.nj_set_option(m, opt, int(value))
            if st != NJ_OK:
                raise NJError(st, "nj_set_option")

    def set_temperature(self, temperature: float):
        for r in range(self.n):
            st = self._lib.nj_set_temperature(self._lib.nj_group_member(self._h, r), float(temperature))
            if st != NJ_OK:
                raise NJError(st, "nj_set_temperature")

    def shards(self, W):
        """Views of a full [V, d] weight as the members' shards."""
        return [W[vb:ve] for vb, ve in self.ranges]

    def verify(self, hidden, W_shards, draft_tokens, draft_probs, gamma, uniforms, accept_len, next_token,
               debug: dict | None = None, stream=None):
        g = np.ascontiguousarray(gamma, np.int32)
        _check_batch(self.cfg, hidden, None, draft_tokens, draft_probs, g, uniforms, accept_len, next_token)
        for r, w in enumerate(W_shards):
            vb, ve = self.ranges[r]
            _dev(w, f"W_shards[{r}]", "bfloat16", ncols=self.cfg.d, min_rows=ve - vb)
        ptrs = (ctypes.c_void_p * self.n)(*[_ptr(w) for w in W_shards])
        dbg = None
        if debug is not None:
            dbg = nj_debug(_ptr(debug.get("lse")), _ptr(debug.get("p_draft")), _ptr(debug.get("mass")),
                           _ptr(debug.get("flags")))
        st = self._lib.nj_group_verify(
            self._h, _stream(stream), _ptr(hidden), ptrs, _ptr(draft_tokens), _ptr(draft_probs),
            int(draft_probs.stride(0)), _ptr(g), _ptr(uniforms), g.shape[0], _ptr(accept_len), _ptr(next_token),
            ctypes.byref(dbg) if dbg is not None else None)
        if st != NJ_OK:
            raise NJError(st, self._lib.nj_group_last_error(self._h).decode())


class Bandit:
    """RAII wrapper of nj_bandit (Nightjar, Algorithm 1 + Eq. 3)."""

    def __init__(self, gamma_max: int, batch_max: int, seed: int = 0, len_buckets=None, batch_buckets=None,
                 cost_ms=None):
        lib = load()
        h = ctypes.c_void_p()
        if cost_ms is not None:
            L = np.ascontiguousarray(len_buckets, np.int32)
            Bb = np.ascontiguousarray(batch_buckets, np.int32)
            C = np.ascontiguousarray(cost_ms, np.float64).reshape(-1)
            self._keep = (L, Bb, C)
            st = lib.nj_bandit_create(gamma_max, batch_max, seed, _ptr(L), L.shape[0], _ptr(Bb), Bb.shape[0],
                                      _ptr(C), ctypes.byref(h))
        else:
            st = lib.nj_bandit_create(gamma_max, batch_max, seed, None, 0, None, 0, None, ctypes.byref(h))
        if st != NJ_OK:
            raise NJError(st, "nj_bandit_create rejected the configuration")
        self._lib, self._h = lib, h
        self.gamma_max, self.batch_max = gamma_max, batch_max

    def close(self):
        if self._h:
            self._lib.nj_bandit_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def select(self, batch_size: int, l_max: int = 0) -> int:
        g = self._lib.nj_select_gamma(self._h, batch_size, l_max)
        if g < 0:
            raise NJError(-g, f"nj_select_gamma({batch_size}, {l_max})")
        return g

    def observe(self, batch_size: int, gamma: int, reward: float):
        st = self._lib.nj_observe(self._h, batch_size, gamma, float(reward))
        if st != NJ_OK:
            raise NJError(st, f"nj_observe({batch_size}, {gamma}, {reward})")

    def score(self, batch_size, gamma_prev, gamma, l_max=0) -> float:
        return self._lib.nj_exploitation_score(self._h, batch_size, gamma_prev, gamma, l_max)

    def prefill_cost_ms(self, l_max, batch_size) -> float:
        return self._lib.nj_prefill_cost_ms(self._h, l_max, batch_size)

    def state(self, batch_size):
        j, H, b, t, bt = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
        st = self._lib.nj_bandit_state(self._h, batch_size, ctypes.byref(j), ctypes.byref(H), ctypes.byref(b),
                                       ctypes.byref(t), ctypes.byref(bt))
        if st != NJ_OK:
            raise NJError(st, "nj_bandit_state")
        return j.value, H.value, b.value, t.value, bt.value

    def arm(self, batch_size, gamma):
        m, n = ctypes.c_double(), ctypes.c_int64()
        st = self._lib.nj_bandit_arm(self._h, batch_size, gamma, ctypes.byref(m), ctypes.byref(n))
        if st != NJ_OK:
            raise NJError(st, "nj_bandit_arm")
        return m.value, n.value

    @property
    def last_gamma(self) -> int:
        return self._lib.nj_bandit_last_gamma(self._h)

    def snapshot(self) -> dict:
        need = ctypes.c_size_t()
        self._lib.nj_bandit_snapshot_json(self._h, None, 0, ctypes.byref(need))
        buf = ctypes.create_string_buffer(need.value)
        st = self._lib.nj_bandit_snapshot_json(self._h, buf, need.value, ctypes.byref(need))
        if st != NJ_OK:
            raise NJError(st, "snapshot")
        return json.loads(buf.value.decode())
