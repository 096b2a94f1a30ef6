"""CPU tests of the drop-in boundary: libafg.so loads, exports exactly the
entry points include/afg.h declares, validates arguments on the host before
touching a device, and has no CPU fallback (compute entry points fail when
no sm_100 device is visible)."""
import ctypes
import os
import re

import pytest

import paper_2603_06731_b200 as afg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    for h in os.listdir(os.path.join(ROOT, "include")):
        if not h.endswith(".h"):
            continue
        text = open(os.path.join(ROOT, "include", h)).read()
        syms |= set(re.findall(r"^AFG_API\s+[\w\s\*]+?\b(afg_\w+)\s*\(", text, re.M))
    return syms


def test_library_builds_and_loads():
    assert os.path.exists(afg.lib_path), "run __graft_entry__.build()"
    L = afg.lib()
    assert L.afg_version().startswith(b"afg")


def test_every_declared_symbol_is_exported():
    L = afg.lib()
    decl = declared_symbols()
    assert len(decl) >= 15
    missing = [s for s in sorted(decl) if not hasattr(L, s)]
    assert not missing, missing


def test_python_binding_covers_header():
    assert declared_symbols() <= set(afg.EXPORTED_SYMBOLS)


def test_argument_validation_is_host_side():
    L = afg.lib()
    st = L.afg_gemm(None, 0, None, 0, None, None, None, 0, 4, 4, 4, 2, 2, 0, 0, None)
    assert st == 1  # AFG_ERR_INVALID_ARG
    assert b"null" in L.afg_last_error()
    p = ctypes.c_void_p(16)
    st = L.afg_gemm(p, 4, p, 4, None, None, p, 4, 4, 4, 0, 2, 2, 0, 0, None)
    assert st == 1 and b"extent" in L.afg_last_error()
    st = L.afg_gemm(p, 4, p, 4, None, None, p, 4, 4, 4, 4, 2, 2, 0, 3, None)  # GELU w/o bias
    assert st == 1 and b"bias" in L.afg_last_error()
    st = L.afg_softmax_lastdim(None, None, 1, 1, 0, 0, None)
    assert st == 1


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    L = afg.lib()
    assert L.afg_device_count() == 0
    p = ctypes.c_void_p(256)
    st = L.afg_gemm(p, 64, p, 64, None, None, p, 64, 64, 64, 64, 2, 2, 0, 0, None)
    assert st == 3  # AFG_ERR_CUDA: no silent CPU path
    with pytest.raises(afg.AfgError):
        afg.ops.gemm(torch.zeros(4, 4), torch.zeros(4, 4))
