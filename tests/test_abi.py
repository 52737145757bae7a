"""The C-ABI library loads and exports every symbol include/nj.h declares,
the product path has no CPU fallback, and the oracle / product code share
nothing (no imports, no includes).  CPU only: no compute calls."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2512_22420_b200 as pkg
from paper_2512_22420_b200 import _build, _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "nj.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nj_[a-z0-9_]+)\s*\(", src)))


def test_library_builds_and_loads():
    path = _build.build()
    assert os.path.exists(path)
    lib = ctypes.CDLL(path)
    assert lib is not None


def test_every_declared_symbol_is_exported():
    lib = ctypes.CDLL(_build.build())
    syms = header_symbols()
    assert len(syms) >= 19
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(syms) == sorted(_lib.EXPORTS)


def test_probes_are_not_in_the_product_library():
    """Measurement probes live in scripts/probes/libnj_probe.so, not libnj.so."""
    out = subprocess.run(["nm", "-D", "--defined-only", _build.build()], capture_output=True, text=True).stdout
    for sym in ("nj_stream_test", "nj_mma_probe", "nj_lmhead_logits_ks", "k_probe_ks", "k_stream_test",
                "k_mma_probe", "k_gemm_acc", "k_gemm_rows"):
        assert sym not in out, sym


def test_sass_is_sm100a_tcgen05():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _build.build()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "UTCHMMA" in out and "UTMALDG" in out and "LDTM" in out


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(pkg.NJError) as e:
        pkg.Verifier(16, 32, 1, 3)
    assert e.value.status == _lib.NJ_ECUDA


def test_oracle_and_product_share_nothing():
    prod = os.path.join(ROOT, "paper_2512_22420_b200")
    orc = os.path.join(ROOT, "oracle")
    for dirpath, _, files in os.walk(prod):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), f
                assert "nj_oracle" not in txt, f
    for f in os.listdir(orc):
        if f.endswith((".py", ".c")):
            txt = open(os.path.join(orc, f)).read()
            assert not re.search(r"^\s*(import|from)\s+paper_2512_22420_b200", txt, re.M), f
            assert not re.search(r"^\s*#\s*include\s+[<\"].*nj[_a-z]*\.(h|cuh)", txt, re.M), f
            assert not re.search(r"CDLL\([^)]*libnj", txt), f


def test_bad_arguments_rejected_before_launch():
    lib = _lib.load()
    assert lib.nj_create(None, None) == _lib.NJ_EINVAL
    cfg = _lib.nj_config(7, 32, 1, 3, 0, None, 0, 32)        # d % 8 != 0
    h = ctypes.c_void_p()
    assert lib.nj_create(ctypes.byref(cfg), ctypes.byref(h)) == _lib.NJ_ESHAPE
    assert b"multiple of 8" in lib.nj_last_error(None)
