"""Torch-facing wrappers over the afg C ABI (device tensors in, device tensors
out). Every function launches on torch's current CUDA stream and raises
AfgError on failure; none has a CPU path."""
from __future__ import annotations

import ctypes

import torch

from . import AfgError, BinOp, DType, Epilogue, Layout, ReduceKind, check, lib

_TORCH2AFG = {torch.float32: DType.F32, torch.float16: DType.F16, torch.bfloat16: DType.BF16}
_AFG2TORCH = {v: k for k, v in _TORCH2AFG.items()}


def afg_dtype(t: torch.dtype) -> DType:
    try:
        return _TORCH2AFG[t]
    except KeyError as e:
        raise AfgError(1, f"unsupported dtype {t}") from e


def torch_dtype(d: DType) -> torch.dtype:
    return _AFG2TORCH[DType(d)]


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise AfgError(1, "afg ops take CUDA tensors (no CPU fallback)")


def gemm(a, b, bias=None, epilogue=Epilogue.NONE, out_dtype=None, b_layout=Layout.B_KN,
         residual=None, out=None):
    """C = epi(A @ B + bias) (+ residual). a [M,K]; b [K,N] (B_KN) or [N,K] (B_NK)."""
    _need_cuda(a, b, bias, residual, out)
    M, K = a.shape
    N = b.shape[1] if b_layout == Layout.B_KN else b.shape[0]
    od = out_dtype or a.dtype
    if out is None:
        out = torch.empty((M, N), dtype=od, device=a.device)
    check(lib().afg_gemm(_ptr(a), a.stride(0), _ptr(b), b.stride(0), _ptr(bias), _ptr(residual),
                         _ptr(out), out.stride(0), M, N, K, afg_dtype(a.dtype), afg_dtype(od),
                         int(b_layout), int(epilogue), _stream()))
    return out


def gemm_i8(a, b_nk, out_mode=0, scale=1.0, out=None):
    """int8 GEMM on tcgen05 kind::i8 (quant repositioning).
    a int8 [M,K], b_nk int8 [N,K]; out_mode 0 -> int32 A.B^T (exact),
    1 -> int8 requantised clamp(round_half_away(acc*scale)), 2 -> float32 acc*scale."""
    _need_cuda(a, b_nk, out)
    if a.dtype != torch.int8 or b_nk.dtype != torch.int8:
        raise AfgError(1, "gemm_i8 takes int8 operands")
    M, K = a.shape
    N = b_nk.shape[0]
    od = {0: torch.int32, 1: torch.int8, 2: torch.float32}[int(out_mode)]
    if out is None:
        out = torch.empty((M, N), dtype=od, device=a.device)
    check(lib().afg_gemm_i8(_ptr(a), a.stride(0), _ptr(b_nk), b_nk.stride(0), _ptr(out),
                            out.stride(0), M, N, K, int(out_mode), float(scale), _stream()))
    return out


def conv2d_nhwc_i8(x, w_ohwi, stride=(1, 1), pad=(0, 0), dil=(1, 1), out_hw=None, out_mode=0,
                   scale=1.0):
    """int8 implicit-GEMM conv (K1c on TMA im2col). x int8 [B,H,W,C], w int8
    [OC,KH,KW,C]; pad = (top, left); out_hw defaults to symmetric padding.
    Returns [B,OH,OW,OC] int32 / int8 / float32 by out_mode (as gemm_i8)."""
    _need_cuda(x, w_ohwi)
    if x.dtype != torch.int8 or w_ohwi.dtype != torch.int8:
        raise AfgError(1, "conv2d_nhwc_i8 takes int8 operands")
    B, H, W, C = x.shape
    OC, KH, KW, _ = w_ohwi.shape
    if out_hw is None:
        out_hw = ((H + 2 * pad[0] - dil[0] * (KH - 1) - 1) // stride[0] + 1,
                  (W + 2 * pad[1] - dil[1] * (KW - 1) - 1) // stride[1] + 1)
    OH, OW = out_hw
    od = {0: torch.int32, 1: torch.int8, 2: torch.float32}[int(out_mode)]
    y = torch.empty((B, OH, OW, OC), dtype=od, device=x.device)
    check(lib().afg_conv2d_nhwc_i8(_ptr(x.contiguous()), _ptr(w_ohwi.contiguous()), _ptr(y), B, H,
                                   W, C, OC, KH, KW, stride[0], stride[1], pad[0], pad[1], dil[0],
                                   dil[1], OH, OW, int(out_mode), float(scale), _stream()))
    return y


def gemm_batched(a, b, out_dtype=None):
    _need_cuda(a, b)
    *bd, M, K = a.shape
    N = b.shape[-1]
    batch = 1
    for d in bd:
        batch *= d
    od = out_dtype or a.dtype
    out = torch.empty((*bd, M, N), dtype=od, device=a.device)
    check(lib().afg_gemm_batched(_ptr(a.contiguous()), _ptr(b.contiguous()), _ptr(out), batch, M,
                                 N, K, afg_dtype(a.dtype), afg_dtype(od), _stream()))
    return out


def softmax(x, out_dtype=None, out=None):
    _need_cuda(x)
    x = x.contiguous()
    od = out_dtype or (out.dtype if out is not None else x.dtype)
    y = out if out is not None else torch.empty(x.shape, dtype=od, device=x.device)
    cols = x.shape[-1]
    check(lib().afg_softmax_lastdim(_ptr(x), _ptr(y), x.numel() // cols, cols, afg_dtype(x.dtype),
                                    afg_dtype(od), _stream()))
    return y


def layernorm_residual(x, residual, gamma, beta, eps=1e-12, sum_out=None, out=None):
    _need_cuda(x, residual, gamma, beta)
    y = out if out is not None else torch.empty_like(x)
    cols = x.shape[-1]
    check(lib().afg_layernorm_residual(_ptr(x), _ptr(residual), _ptr(gamma), _ptr(beta), _ptr(y),
                                       _ptr(sum_out), x.numel() // cols, cols, eps,
                                       afg_dtype(x.dtype), _stream()))
    return y


def elementwise(a, b, op: BinOp, out_dtype=None, b_period=0):
    _need_cuda(a, b)
    od = out_dtype or a.dtype
    out = torch.empty(a.shape, dtype=od, device=a.device)
    check(lib().afg_elementwise(_ptr(a), _ptr(b), _ptr(out), a.numel(), b_period, int(op),
                                afg_dtype(a.dtype), afg_dtype(b.dtype if b is not None else a.dtype),
                                afg_dtype(od), _stream()))
    return out


def reduce_lastdim(x, kind: ReduceKind, out_dtype=None):
    _need_cuda(x)
    od = out_dtype or x.dtype
    cols = x.shape[-1]
    out = torch.empty(x.shape[:-1], dtype=od, device=x.device)
    check(lib().afg_reduce_lastdim(_ptr(x), _ptr(out), x.numel() // cols, cols, int(kind),
                                   afg_dtype(x.dtype), afg_dtype(od), _stream()))
    return out


def convert(x, dtype):
    _need_cuda(x)
    y = torch.empty(x.shape, dtype=dtype, device=x.device)
    check(lib().afg_convert(_ptr(x), _ptr(y), x.numel(), afg_dtype(x.dtype), afg_dtype(dtype),
                            _stream()))
    return y


def transpose(x, perm):
    _need_cuda(x)
    x = x.contiguous()
    shape = (ctypes.c_int64 * x.dim())(*x.shape)
    p = (ctypes.c_int64 * x.dim())(*perm)
    y = torch.empty([x.shape[i] for i in perm], dtype=x.dtype, device=x.device)
    check(lib().afg_transpose(_ptr(x), _ptr(y), x.dim(), ctypes.cast(shape, ctypes.c_void_p),
                              ctypes.cast(p, ctypes.c_void_p), afg_dtype(x.dtype), _stream()))
    return y


def fill_uniform(shape, seed, lo=0.0, hi=1.0, dtype=torch.float32, device="cuda"):
    """Device-side makeRandomTensor (interp.cpp:817-844): seed is the stream
    state s0 = seed ^ std::hash<std::string>(id) (see oracle.stream_seed)."""
    x = torch.empty(shape, dtype=dtype, device=device)
    check(lib().afg_fill_uniform(_ptr(x), x.numel(), ctypes.c_uint64(seed & (2**64 - 1)), lo, hi,
                                 afg_dtype(dtype), _stream()))
    return x


def conv2d_nhwc(x, w_ohwi, bias=None, stride=(1, 1), pad=(0, 0), dilation=(1, 1),
                epilogue=Epilogue.NONE, out_hw=None):
    """x [B,H,W,C], w [OC,KH,KW,C] -> y [B,OH,OW,OC]; pad = (top, left)."""
    _need_cuda(x, w_ohwi, bias)
    B, H, W, C = x.shape
    OC, KH, KW, _ = w_ohwi.shape
    if out_hw is None:
        OH = (H + 2 * pad[0] - dilation[0] * (KH - 1) - 1) // stride[0] + 1
        OW = (W + 2 * pad[1] - dilation[1] * (KW - 1) - 1) // stride[1] + 1
    else:
        OH, OW = out_hw
    y = torch.empty((B, OH, OW, OC), dtype=x.dtype, device=x.device)
    check(lib().afg_conv2d_nhwc(_ptr(x), _ptr(w_ohwi), _ptr(bias), _ptr(y), B, H, W, C, OC, KH, KW,
                                stride[0], stride[1], pad[0], pad[1], dilation[0], dilation[1],
                                OH, OW, afg_dtype(x.dtype), int(epilogue), _stream()))
    return y


def conv2d_nchw(x, w, stride=(1, 1), dilation=(1, 1), pad=(0, 0), transposed=False,
                out_hw=None, out_dtype=None):
    _need_cuda(x, w)
    B, C, H, W = x.shape
    OC = w.shape[1] if transposed else w.shape[0]
    KH, KW = w.shape[2], w.shape[3]
    OH, OW = out_hw
    od = out_dtype or x.dtype
    y = torch.empty((B, OC, OH, OW), dtype=od, device=x.device)
    check(lib().afg_conv2d_nchw(_ptr(x), _ptr(w), _ptr(y), B, C, H, W, OC, KH, KW, stride[0],
                                stride[1], dilation[0], dilation[1], pad[0], pad[1],
                                int(transposed), OH, OW, afg_dtype(x.dtype), afg_dtype(od),
                                _stream()))
    return y


def conv_pack_filter(w_oihw):
    _need_cuda(w_oihw)
    OC, C, KH, KW = w_oihw.shape
    out = torch.empty((OC, KH, KW, C), dtype=w_oihw.dtype, device=w_oihw.device)
    check(lib().afg_conv_pack_filter(_ptr(w_oihw.contiguous()), _ptr(out), OC, C, KH, KW,
                                     afg_dtype(w_oihw.dtype), _stream()))
    return out


def attention(q, k, v, bias=None, scale=1.0, causal=False, out_dtype=None, out=None):
    """o = softmax(scale q k^T + bias [+causal]) v; q,k,v [B,H,N,D]."""
    _need_cuda(q, k, v, bias)
    B, H, Nq, D = q.shape
    Nk = k.shape[2]
    od = out_dtype or (out.dtype if out is not None else q.dtype)
    o = out if out is not None else torch.empty((B, H, Nq, D), dtype=od, device=q.device)
    check(lib().afg_attention_fwd(_ptr(q), _ptr(k), _ptr(v), _ptr(bias), _ptr(o), B, H, Nq, Nk, D,
                                  scale, int(causal), afg_dtype(q.dtype), afg_dtype(od), _stream()))
    return o
