"""oracle - TEST INFRASTRUCTURE ONLY.

CPU checkers for the afg kernels. Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu_baseline / ``--impl reference`` arm may import this
package, and only as the checker / the timed reference CPU path; the product
(``paper_2603_06731_b200``) never does.

Two layers:
  * ``liboracle.so`` (oracle.c): plain-C restatement of the reference
    arithmetic, each function citing the reference file:line it follows.
  * ``_ref/libafref.so``: the UNMODIFIED reference library (AffineForge,
    /root/reference/proj) compiled by oracle/Makefile, driven through
    ref_shim.cpp: af::interpret, oracle::evalGraphReference,
    makeRandomInputs, roundToType, compareTensors.
The restatement is pinned against the reference tests' known answers
(tests/golden/) and against _ref (tests/test_oracle.py).
"""
from __future__ import annotations

import ctypes
import json
import os
import struct

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(_HERE, "liboracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libafref.so")

# element-type codes (oracle.c): the reference's ElementType order + BF16
F32, F16, I8, I32, BF16, F64 = 0, 1, 2, 3, 10, 11
TYPE_CODES = {"f32": F32, "f16": F16, "i8": I8, "i32": I32, "bf16": BF16}
# epilogue codes (include/afg.h)
EPI_NONE, EPI_BIAS, EPI_RELU, EPI_GELU_TANH, EPI_GELU_ERF = range(5)
# tolerance profiles (interp.cpp:106-118)
TOL = {"F32": 1e-6, "F16Fragment": 2e-3, "AttentionRR": 1e-3, "Int": 0.0}

_D = ctypes.POINTER(ctypes.c_double)
_L = ctypes.POINTER(ctypes.c_int64)
_I64 = ctypes.c_int64
_i = ctypes.c_int

_orc = None
_ref = None


def _dp(a):
    return a.ctypes.data_as(_D) if a is not None else None


def _lp(a):
    return a.ctypes.data_as(_L) if a is not None else None


def lib():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"{ORACLE_SO} not built (make -C oracle)")
        L = ctypes.CDLL(ORACLE_SO)
        L.orc_round_f16.restype = ctypes.c_double
        L.orc_round_f16.argtypes = [ctypes.c_double]
        L.orc_round_bf16.restype = ctypes.c_double
        L.orc_round_bf16.argtypes = [ctypes.c_double]
        L.orc_round_to_type.restype = ctypes.c_double
        L.orc_round_to_type.argtypes = [ctypes.c_double, _i]
        L.orc_round_array.argtypes = [_D, _I64, _i]
        L.orc_std_hash.restype = ctypes.c_uint64
        L.orc_std_hash.argtypes = [ctypes.c_char_p]
        L.orc_stream_seed.restype = ctypes.c_uint64
        L.orc_stream_seed.argtypes = [ctypes.c_char_p, ctypes.c_uint64]
        L.orc_random_tensor.argtypes = [_D, _I64, ctypes.c_char_p, ctypes.c_uint64,
                                        ctypes.c_double, ctypes.c_double, _i]
        L.orc_random_stream.argtypes = [_D, _I64, ctypes.c_uint64, ctypes.c_double, ctypes.c_double]
        L.orc_matmul.argtypes = [_D, _D, _D, _D, _I64, _I64, _I64, _i, _i, _i, _i, _i, _L, _I64, _i]
        L.orc_batch_matmul.argtypes = [_D, _D, _D, _I64, _I64, _I64, _I64]
        L.orc_conv_geometry.argtypes = [_I64] * 8 + [_i, _i, _L]
        L.orc_conv_nchw.argtypes = [_D, _D, _D] + [_I64] * 13 + [_i, _I64, _I64, _i]
        L.orc_conv_nhwc.argtypes = [_D, _D, _D, _D] + [_I64] * 15 + [_i, _i, _L, _I64, _i]
        L.orc_attention.argtypes = [_D, _D, _D, _D, _D, _I64, _I64, _I64, _I64, ctypes.c_double,
                                    _i, _L, _I64, _i]
        L.orc_softmax.argtypes = [_D, _D, _I64, _I64]
        L.orc_layernorm.argtypes = [_D, _D, _D, _D, _D, _D, _I64, _I64, ctypes.c_double]
        L.orc_compare.restype = _i
        L.orc_compare.argtypes = [_D, _D, _I64, ctypes.c_double, _D, _D, _L]
        _orc = L
    return _orc


def threads():
    return max(1, os.cpu_count() or 1)


def f64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


# ------------------------------------------------------------- rounding ---

def round_to(x, t):
    """roundToType (interp.cpp:88-104) elementwise; t in F32/F16/I8/I32/BF16."""
    a = f64(x).copy()
    lib().orc_round_array(_dp(a), a.size, t)
    return a


def round_f16(v: float) -> float:
    return lib().orc_round_f16(v)


# ------------------------------------------------------------------ RNG ---

def std_hash(s: str) -> int:
    return lib().orc_std_hash(s.encode())


def stream_seed(buffer_id: str, seed: int) -> int:
    """s0 = seed ^ std::hash<std::string>(id) (interp.cpp:833); the device
    generator afg_fill_uniform(seed=s0) reproduces the same stream."""
    return lib().orc_stream_seed(buffer_id.encode(), seed & (2**64 - 1))


def random_tensor(shape, buffer_id: str, seed: int, lo=0.0, hi=1.0, is_int=False):
    """makeRandomTensor (interp.cpp:817-844); buffer_id as in lowered programs ('%a')."""
    n = int(np.prod(shape)) if len(shape) else 1
    out = np.empty(n, dtype=np.float64)
    lib().orc_random_tensor(_dp(out), n, buffer_id.encode(), seed & (2**64 - 1), lo, hi,
                            int(is_int))
    return out.reshape(shape)


def random_stream(shape, s0: int, lo=0.0, hi=1.0):
    """Draws of the splitmix64 stream with state s0 (what afg_fill_uniform
    generates on the device for seed s0)."""
    n = int(np.prod(shape)) if len(shape) else 1
    out = np.empty(n, dtype=np.float64)
    lib().orc_random_stream(_dp(out), n, s0 & (2**64 - 1), lo, hi)
    return out.reshape(shape)


# --------------------------------------------------------------- matmul ---

def matmul(A, B, bias=None, epi=EPI_NONE, out_t=F32, acc_t=F32, b_nk=False, interp=False,
           rows=None, nthreads=None):
    A = f64(A)
    B = f64(B)
    M, K = A.shape
    N = B.shape[0] if b_nk else B.shape[1]
    rows_a = None if rows is None else np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    n_out = M if rows_a is None else len(rows_a)
    C = np.empty((n_out, N), dtype=np.float64)
    bias_a = None if bias is None else f64(bias)
    lib().orc_matmul(_dp(A), _dp(B), _dp(bias_a), _dp(C), M, N, K, epi, acc_t, out_t,
                     int(b_nk), int(interp), _lp(rows_a), 0 if rows_a is None else len(rows_a),
                     nthreads or threads())
    return C


def batch_matmul(A, B):
    A = f64(A)
    B = f64(B)
    *bd, M, K = A.shape
    N = B.shape[-1]
    batch = int(np.prod(bd)) if bd else 1
    C = np.empty((*bd, M, N), dtype=np.float64)
    lib().orc_batch_matmul(_dp(A), _dp(B), _dp(C), batch, M, N, K)
    return C


# ------------------------------------------------------------- int8 GEMM ---

def quantize(x, scale):
    """The interpreter's `quant`: clamp(round_half_away(x / scale), -128, 127)
    (test_interp.cpp:286-307 KAT; SPEC.md:531-572 QuantScheme)."""
    y = np.asarray(x, dtype=np.float64) / np.float64(scale)
    return np.clip(np.sign(y) * np.floor(np.abs(y) + 0.5), -128, 127)


def matmul_i8(A, B_nk, mode=0, scale=1.0, rows=None):
    """int8 x int8 -> int32 matmul as the reference evaluates an i8 matmul
    graph (lowerMatmul nest, frontend.cpp:679-733; double arithmetic exact
    for |sum| < 2^53, interp.cpp:502-561; I32 store = nearbyint + saturate,
    interp.cpp:25-104), with B given as [N, K]. mode 1 requantises the
    accumulator with round half away from zero and saturation (the `quant`
    op), mode 2 dequantises to f32; scale is the f32 the C ABI receives,
    applied in double."""
    A = np.asarray(A, dtype=np.int64)
    if rows is not None:
        A = A[np.asarray(rows)]
    acc = np.clip(A @ np.asarray(B_nk, dtype=np.int64).T, -2**31, 2**31 - 1)
    if mode == 0:
        return acc.astype(np.int32)
    x = acc.astype(np.float64) * np.float64(np.float32(scale))
    if mode == 1:
        return np.clip(np.sign(x) * np.floor(np.abs(x) + 0.5), -128, 127).astype(np.int8)
    return x.astype(np.float32)


def conv_i8(x, w_ohwi, stride=(1, 1), pad=(0, 0), dil=(1, 1), out_hw=None, mode=0, scale=1.0):
    """Exact integer NHWC conv (the reference's i8 conv graph nest,
    frontend.cpp:752-970, evaluated in double = exact integers), i32 result,
    then matmul_i8's requantise / dequantise. x [B,H,W,C], w [OC,KH,KW,C]."""
    x = np.asarray(x, dtype=np.int64)
    w = np.asarray(w_ohwi, dtype=np.int64)
    B, H, W, C = x.shape
    OC, KH, KW, _ = w.shape
    if out_hw is None:
        out_hw = ((H + 2 * pad[0] - dil[0] * (KH - 1) - 1) // stride[0] + 1,
                  (W + 2 * pad[1] - dil[1] * (KW - 1) - 1) // stride[1] + 1)
    OH, OW = out_hw
    hp = max(H + pad[0], (OH - 1) * stride[0] + (KH - 1) * dil[0] + 1)
    wp = max(W + pad[1], (OW - 1) * stride[1] + (KW - 1) * dil[1] + 1)
    xp = np.zeros((B, hp, wp, C), dtype=np.int64)
    xp[:, pad[0]:pad[0] + H, pad[1]:pad[1] + W, :] = x
    acc = np.zeros((B, OH, OW, OC), dtype=np.int64)
    for ky in range(KH):
        for kx in range(KW):
            ys, xs = ky * dil[0], kx * dil[1]
            patch = xp[:, ys:ys + (OH - 1) * stride[0] + 1:stride[0],
                       xs:xs + (OW - 1) * stride[1] + 1:stride[1], :]
            acc += np.einsum("bhwc,oc->bhwo", patch, w[:, ky, kx, :])
    acc = np.clip(acc, -2**31, 2**31 - 1)
    if mode == 0:
        return acc.astype(np.int32)
    v = acc.astype(np.float64) * np.float64(np.float32(scale))
    if mode == 1:
        return np.clip(np.sign(v) * np.floor(np.abs(v) + 0.5), -128, 127).astype(np.int8)
    return v.astype(np.float32)


# ----------------------------------------------------------------- conv ---

def conv_geometry(inH, inW, kH, kW, stride=(1, 1), dil=(1, 1), same=False, transposed=False):
    out = np.zeros(4, dtype=np.int64)
    lib().orc_conv_geometry(inH, inW, kH, kW, stride[0], stride[1], dil[0], dil[1], int(same),
                            int(transposed), _lp(out))
    return tuple(int(v) for v in out)


def conv_nchw(x, w, stride=(1, 1), dil=(1, 1), pad=(0, 0), transposed=False, out_hw=None,
              out_t=F32):
    x = f64(x)
    w = f64(w)
    B, C, H, W = x.shape
    OC = w.shape[1] if transposed else w.shape[0]
    KH, KW = w.shape[2], w.shape[3]
    OH, OW = out_hw
    y = np.empty((B, OC, OH, OW), dtype=np.float64)
    lib().orc_conv_nchw(_dp(x), _dp(w), _dp(y), B, C, H, W, OC, KH, KW, stride[0], stride[1],
                        dil[0], dil[1], pad[0], pad[1], int(transposed), OH, OW, out_t)
    return y


def conv_nhwc(x, w_ohwi, bias=None, stride=(1, 1), pad=(0, 0), dil=(1, 1), out_hw=None,
              epi=EPI_NONE, out_t=F32, images=None, nthreads=None):
    x = f64(x)
    w = f64(w_ohwi)
    B, H, W, C = x.shape
    OC, KH, KW, _ = w.shape
    if out_hw is None:
        OH = (H + 2 * pad[0] - dil[0] * (KH - 1) - 1) // stride[0] + 1
        OW = (W + 2 * pad[1] - dil[1] * (KW - 1) - 1) // stride[1] + 1
    else:
        OH, OW = out_hw
    img = None if images is None else np.ascontiguousarray(np.asarray(images, dtype=np.int64))
    nb = B if img is None else len(img)
    y = np.empty((nb, OH, OW, OC), dtype=np.float64)
    b = None if bias is None else f64(bias)
    lib().orc_conv_nhwc(_dp(x), _dp(w), _dp(b), _dp(y), B, H, W, C, OC, KH, KW, stride[0],
                        stride[1], pad[0], pad[1], dil[0], dil[1], OH, OW, epi, out_t, _lp(img),
                        0 if img is None else len(img), nthreads or threads())
    return y


# ------------------------------------------------------------ attention ---

def attention(q, k, v, bias=None, scale=1.0, causal=False, heads=None, nthreads=None):
    """q,k,v [B,H,N,D] -> o [B,H,N,D] (or [len(heads),N,D] for a subset of
    flattened (b,h) indices)."""
    q = f64(q)
    k = f64(k)
    v = f64(v)
    B, H, Nq, D = q.shape
    Nk = k.shape[2]
    hs = None if heads is None else np.ascontiguousarray(np.asarray(heads, dtype=np.int64))
    nh = B * H if hs is None else len(hs)
    o = np.empty((nh, Nq, D), dtype=np.float64)
    b = None if bias is None else f64(bias)
    lib().orc_attention(_dp(q), _dp(k), _dp(v), _dp(b), _dp(o), B * H, Nq, Nk, D, scale,
                        int(causal), _lp(hs), 0 if hs is None else len(hs), nthreads or threads())
    return o.reshape(B, H, Nq, D) if hs is None else o


# -------------------------------------------------------------- chains ---

def softmax(x):
    x = f64(x)
    y = np.empty_like(x)
    cols = x.shape[-1]
    lib().orc_softmax(_dp(x), _dp(y), x.size // cols, cols)
    return y


def layernorm(x, res, gamma, beta, eps):
    x = f64(x)
    r = None if res is None else f64(res)
    g = f64(gamma)
    b = f64(beta)
    y = np.empty_like(x)
    s = np.empty_like(x)
    cols = x.shape[-1]
    lib().orc_layernorm(_dp(x), _dp(r), _dp(g), _dp(b), _dp(y), _dp(s), x.size // cols, cols, eps)
    return y, s


def compare(a, b, tol):
    """compareTensors (interp.cpp:698-730). Returns (passed, max_abs, max_rel, worst)."""
    a = f64(a).ravel()
    b = f64(b).ravel()
    if a.shape != b.shape:
        raise ValueError("compare: shape mismatch")
    ma = ctypes.c_double()
    mr = ctypes.c_double()
    w = ctypes.c_int64()
    ok = lib().orc_compare(_dp(a), _dp(b), a.size, tol, ctypes.byref(ma), ctypes.byref(mr),
                           ctypes.byref(w))
    return bool(ok), ma.value, mr.value, w.value


# ============================================================ reference ===

class RefError(RuntimeError):
    pass


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not ref_available():
            raise RefError(f"{REF_SO} not built (make -C oracle ref, needs /root/reference)")
        L = ctypes.CDLL(REF_SO)
        L.afref_run.restype = ctypes.c_void_p
        L.afref_run.argtypes = [ctypes.c_char_p, _i, ctypes.POINTER(ctypes.c_char_p),
                                ctypes.POINTER(_D), _L, _i, ctypes.c_char_p, _i]
        L.afref_random_inputs.restype = ctypes.c_void_p
        L.afref_random_inputs.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_double,
                                          ctypes.c_double, ctypes.c_char_p, _i]
        for n in ("afref_result_count",):
            getattr(L, n).restype = _i
            getattr(L, n).argtypes = [ctypes.c_void_p]
        L.afref_result_name.restype = ctypes.c_char_p
        L.afref_result_name.argtypes = [ctypes.c_void_p, _i]
        L.afref_result_rank.restype = _i
        L.afref_result_rank.argtypes = [ctypes.c_void_p, _i]
        L.afref_result_dim.restype = _I64
        L.afref_result_dim.argtypes = [ctypes.c_void_p, _i, _i]
        L.afref_result_type.restype = _i
        L.afref_result_type.argtypes = [ctypes.c_void_p, _i]
        L.afref_result_numel.restype = _I64
        L.afref_result_numel.argtypes = [ctypes.c_void_p, _i]
        L.afref_result_data.restype = _D
        L.afref_result_data.argtypes = [ctypes.c_void_p, _i]
        L.afref_result_metrics.restype = ctypes.c_char_p
        L.afref_result_metrics.argtypes = [ctypes.c_void_p]
        L.afref_free.argtypes = [ctypes.c_void_p]
        L.afref_round_to_type.restype = ctypes.c_double
        L.afref_round_to_type.argtypes = [ctypes.c_double, _i]
        L.afref_round_to_f16.restype = ctypes.c_double
        L.afref_round_to_f16.argtypes = [ctypes.c_double]
        L.afref_std_hash.restype = ctypes.c_uint64
        L.afref_std_hash.argtypes = [ctypes.c_char_p]
        L.afref_compare.restype = _i
        L.afref_compare.argtypes = [_D, _D, _I64, _i, _D, _D, _L]
        L.afref_conv_geometry.argtypes = [_I64] * 8 + [_i, _i, _L]
        _ref = L
    return _ref


def _unpack(L, h):
    out = {}
    try:
        for i in range(L.afref_result_count(h)):
            name = L.afref_result_name(h, i).decode()
            rank = L.afref_result_rank(h, i)
            shape = tuple(L.afref_result_dim(h, i, d) for d in range(rank))
            n = L.afref_result_numel(h, i)
            p = L.afref_result_data(h, i)
            arr = np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0)
            out[name] = arr.reshape(shape)
    finally:
        pass
    return out


def ref_run(graph_json: str, inputs: dict, which: str = "interpret", want_metrics=False):
    """Runs the unmodified reference on a graph: which = "interpret"
    (lowerGraphToAffine + af::interpret) or "oracle" (evalGraphReference).
    inputs: {tensor id (no '%'): array}. Returns {"%id": array}."""
    L = ref_lib()
    names = list(inputs)
    arrs = [f64(inputs[n]).ravel() for n in names]
    c_names = (ctypes.c_char_p * len(names))(*[n.encode() for n in names])
    c_data = (_D * len(names))(*[_dp(a) for a in arrs])
    c_numel = (ctypes.c_int64 * len(names))(*[a.size for a in arrs])
    err = ctypes.create_string_buffer(2048)
    h = L.afref_run(graph_json.encode() if isinstance(graph_json, str) else graph_json,
                    len(names), c_names, c_data, c_numel, 0 if which == "interpret" else 1, err,
                    2048)
    if not h:
        raise RefError(err.value.decode())
    try:
        out = _unpack(L, h)
        metrics = L.afref_result_metrics(h).decode() if want_metrics else None
    finally:
        L.afref_free(h)
    return (out, json.loads(metrics)) if want_metrics else out


def ref_random_inputs(graph_json: str, seed: int, lo=0.0, hi=1.0):
    L = ref_lib()
    err = ctypes.create_string_buffer(2048)
    h = L.afref_random_inputs(graph_json.encode(), seed & (2**64 - 1), lo, hi, err, 2048)
    if not h:
        raise RefError(err.value.decode())
    try:
        return _unpack(L, h)
    finally:
        L.afref_free(h)


def ref_compare(a, b, profile: str):
    L = ref_lib()
    a = f64(a).ravel()
    b = f64(b).ravel()
    prof = {"F32": 0, "F16Fragment": 1, "AttentionRR": 2, "Int": 3}[profile]
    ma = ctypes.c_double()
    mr = ctypes.c_double()
    w = ctypes.c_int64()
    ok = L.afref_compare(_dp(a), _dp(b), a.size, prof, ctypes.byref(ma), ctypes.byref(mr),
                         ctypes.byref(w))
    return bool(ok), ma.value, mr.value, w.value


# ---------------------------------------------------------- graph utils ---

def graph_inputs(graph: dict):
    """Tensor ids never produced by an op (TensorGraph::inputIds, frontend.cpp:29-38)."""
    produced = {op["output"] for op in graph["ops"]}
    return [t["id"] for t in graph["tensors"] if t["id"] not in produced]


def random_graph_inputs(graph: dict, seed: int, lo=0.0, hi=1.0):
    """makeRandomInputs (interp.cpp:846-853) for the lowered graph's input
    buffers ('%' + id), restated: {id: array}."""
    decl = {t["id"]: t for t in graph["tensors"]}
    out = {}
    for tid in graph_inputs(graph):
        t = decl[tid]
        dt = t.get("dtype", "f32")
        out[tid] = random_tensor(tuple(t["shape"]), "%" + tid, seed, lo, hi,
                                 is_int=dt in ("i8", "i32"))
    return out


def bits_f32(v: float) -> int:
    return struct.unpack("<I", struct.pack("<f", v))[0]
