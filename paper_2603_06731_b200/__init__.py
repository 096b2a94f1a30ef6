"""paper_2603_06731_b200 - B200-native (sm_100a) operator kernels for the
AffineForge / PolyBlocks graph API.

The product is the C-ABI shared library ``libafg.so`` (declared in
``include/afg.h``) built from ``csrc/``: hand-written tcgen05/TMA kernels for
matmul (+bias/ReLU/GELU epilogue), implicit-GEMM convolution, fused
attention and the memory-bound softmax / layernorm chains, plus the C++ graph
executor that mirrors ``af::interpret`` (``csrc/graph.cpp``).

This module is a thin ctypes binding used by the tests and ``bench.py``.
PyTorch is used only for device memory and streams (plumbing). There is no
CPU fallback: importing works anywhere (so the CPU test suite can check the
exported symbols), but every compute call raises ``AfgError`` when the
library is missing or no sm_100 device is visible.
"""
from __future__ import annotations

import ctypes
import os
from enum import IntEnum

__all__ = [
    "AfgError", "DType", "Epilogue", "Layout", "BinOp", "ReduceKind", "lib", "lib_path",
    "load", "EXPORTED_SYMBOLS",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# AFG_LIB_PATH: load another build of the same library (A/B measurements)
lib_path = os.environ.get("AFG_LIB_PATH") or os.path.join(_HERE, "libafg.so")


class AfgError(RuntimeError):
    """Raised for any non-OK afg_status (message from afg_last_error())."""

    def __init__(self, status: int, message: str):
        super().__init__(f"afg status {status}: {message}")
        self.status = status


class DType(IntEnum):
    F32 = 0
    F16 = 1
    BF16 = 2


class Epilogue(IntEnum):
    NONE = 0
    BIAS = 1
    BIAS_RELU = 2
    BIAS_GELU_TANH = 3
    BIAS_GELU_ERF = 4


class Layout(IntEnum):
    B_KN = 0
    B_NK = 1


class BinOp(IntEnum):
    ADD = 0
    SUB = 1
    MUL = 2
    MAX = 3
    EXP = 4


class ReduceKind(IntEnum):
    SUM = 0
    MAX = 1
    MAXABS = 2


_P = ctypes.c_void_p
_I = ctypes.c_int64
_i = ctypes.c_int
_f = ctypes.c_float

# name -> (restype, argtypes); must match include/afg.h
_SIGS = {
    "afg_last_error": (ctypes.c_char_p, []),
    "afg_version": (ctypes.c_char_p, []),
    "afg_device_count": (_i, []),
    "afg_launch_count": (ctypes.c_uint64, []),
    "afg_gemm": (_i, [_P, _I, _P, _I, _P, _P, _P, _I, _I, _I, _I, _i, _i, _i, _i, _P]),
    "afg_gemm_batched": (_i, [_P, _P, _P, _I, _I, _I, _I, _i, _i, _P]),
    "afg_conv2d_nhwc": (_i, [_P, _P, _P, _P] + [_I] * 15 + [_i, _i, _P]),
    "afg_conv2d_nhwc_ex": (_i, [_P, _P, _P, _P] + [_I] * 15 + [_i, _i, _i, _P]),
    "afg_conv2d_nchw": (_i, [_P, _P, _P] + [_I] * 13 + [_i, _I, _I, _i, _i, _P]),
    "afg_conv_pack_filter": (_i, [_P, _P, _I, _I, _I, _I, _i, _P]),
    "afg_attention_fwd": (_i, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _f, _i, _i, _i, _P]),
    "afg_attention_fwd_strided": (_i, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _f, _i, _i, _i,
                                       _P, _P, _P, _P, _P]),
    "afg_encoder_layer_workspace": (ctypes.c_size_t, [_I, _I, _I, _I, _i]),
    "afg_encoder_layer_fwd": (_i, [_P, _P, _I, _I, _I, _I, _I] + [_P] * 12 + [_f, _i, _P,
                                                                             ctypes.c_size_t, _P]),
    "afg_softmax_lastdim": (_i, [_P, _P, _I, _I, _i, _i, _P]),
    "afg_layernorm_residual": (_i, [_P, _P, _P, _P, _P, _P, _I, _I, _f, _i, _P]),
    "afg_elementwise": (_i, [_P, _P, _P, _I, _I, _i, _i, _i, _i, _P]),
    "afg_reduce_lastdim": (_i, [_P, _P, _I, _I, _i, _i, _i, _P]),
    "afg_epilogue_apply": (_i, [_P, _P, _P, _P, _I, _I, _I, _i, _i, _i, _P]),
    "afg_convert": (_i, [_P, _P, _I, _i, _i, _P]),
    "afg_transpose": (_i, [_P, _P, _i, _P, _P, _i, _P]),
    "afg_fill_uniform": (_i, [_P, _I, ctypes.c_uint64, _f, _f, _i, _P]),
    "afg_broadcast_in_dim": (_i, [_P, _P, _i, _P, _i, _P, _P, _i, _i, _P]),
    "afg_quantize": (_i, [_P, _P, _I, _f, _i, _i, _i, _P]),
    "afg_gemm_i8": (_i, [_P, _I, _P, _I, _P, _I, _I, _I, _I, _i, _f, _P]),
    "afg_conv2d_nhwc_i8": (_i, [_P, _P, _P] + [_I] * 15 + [_i, _f, _P]),
    "afg_comm_unique_id": (_i, [_P]),
    "afg_comm_init_rank": (_i, [ctypes.POINTER(_P), _i, _P, _i]),
    "afg_comm_init_all": (_i, [ctypes.POINTER(_P), _i, ctypes.POINTER(_i)]),
    "afg_comm_destroy": (_i, [_P]),
    "afg_gemm_splitk_workspace": (ctypes.c_size_t, [_I, _I, _i, _i]),
    "afg_gemm_splitk": (_i, [_P, _I, _P, _I, _P, _P, _I, _I, _I, _I, _i, _i, _i, _i, _P, _i, _P,
                             ctypes.c_size_t, _P]),
    "afg_group_create": (_i, [_i, ctypes.POINTER(_i), ctypes.POINTER(_P)]),
    "afg_group_destroy": (None, [_P]),
    "afg_group_size": (_i, [_P]),
    "afg_group_run": (_i, [_P, _P, _P]),
    "afg_graph_run": (_i, [ctypes.c_char_p, _i, ctypes.POINTER(ctypes.c_char_p),
                           ctypes.POINTER(ctypes.POINTER(ctypes.c_double)),
                           ctypes.POINTER(_I), _i, _P, ctypes.POINTER(_P)]),
    "afg_graph_run_sharded": (_i, [ctypes.c_char_p, _i, ctypes.POINTER(ctypes.c_char_p),
                                   ctypes.POINTER(ctypes.POINTER(ctypes.c_double)),
                                   ctypes.POINTER(_I), _i, _i, ctypes.POINTER(_i), _I,
                                   ctypes.POINTER(_P)]),
    "afg_graph_result_count": (_i, [_P]),
    "afg_graph_result_name": (ctypes.c_char_p, [_P, _i]),
    "afg_graph_result_rank": (_i, [_P, _i]),
    "afg_graph_result_dim": (_I, [_P, _i, _i]),
    "afg_graph_result_numel": (_I, [_P, _i]),
    "afg_graph_result_data": (ctypes.POINTER(ctypes.c_double), [_P, _i]),
    "afg_graph_result_plan": (ctypes.c_char_p, [_P]),
    "afg_graph_result_free": (None, [_P]),
    "afg_graph_check_json": (_i, [ctypes.c_char_p]),
}
EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None


def load(path: str | None = None):
    """Loads libafg.so (once). Raises AfgError if it is missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or lib_path
    if not os.path.exists(p):
        raise AfgError(-1, f"{p} not built (run `make lib` or __graft_entry__.build())")
    L = ctypes.CDLL(p)
    for name, (res, args) in _SIGS.items():
        fn = getattr(L, name, None)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = L
    return L


def lib():
    return load()


def check(status: int) -> None:
    if status != 0:
        msg = lib().afg_last_error().decode(errors="replace")
        raise AfgError(status, msg)


def launch_count() -> int:
    return int(lib().afg_launch_count())


from . import ops  # noqa: E402,F401  (torch-facing wrappers)
from . import graph  # noqa: E402,F401  (graph executor binding)
