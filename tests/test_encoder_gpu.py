"""GPU parity of the BERT-base encoder layer composition
(afg_encoder_layer_fwd: QKV GEMM -> strided fused attention -> out-proj +
residual -> LN -> GELU FFN -> FFN2 + residual -> LN) against the oracle
composed from the restated reference ops, with every intermediate rounded to
bf16 at the same points as the kernels store it.

Tolerance: 2^-5 in the reference's max(|a|,|b|,1) rule for the final bf16
output (a few bf16 ulps: single-ulp rounding flips in intermediates propagate
through two layernorms); intermediates are not observable."""
import ctypes

import numpy as np
import pytest
import torch

import oracle as O
from paper_2603_06731_b200 import check as afg_check
from paper_2603_06731_b200 import lib
from tests.gpu_util import check, seeded, to_host

pytestmark = pytest.mark.gpu


def oracle_bert(xh, p, B, S, hd, H, ffn):
    """The layer composed from the restated ops, bf16 stores where the kernels
    store (x [B*S, hd] for B whole sequences)."""
    D = hd // H
    T = B * S
    bfr = lambda a: O.round_to(a, O.BF16)  # noqa: E731
    qkv = bfr(O.matmul(xh, p["wqkv"], p["bqkv"], epi=O.EPI_BIAS, out_t=O.F64))
    q = qkv[:, :hd].reshape(B, S, H, D).transpose(0, 2, 1, 3)
    k = qkv[:, hd:2 * hd].reshape(B, S, H, D).transpose(0, 2, 1, 3)
    v = qkv[:, 2 * hd:].reshape(B, S, H, D).transpose(0, 2, 1, 3)
    att = bfr(O.attention(q, k, v, scale=D ** -0.5).transpose(0, 2, 1, 3).reshape(T, hd))
    y1 = bfr(O.matmul(att, p["wo"], p["bo"], epi=O.EPI_BIAS, out_t=O.F64) + xh)
    h1 = bfr(O.layernorm(y1, None, p["g1"], p["be1"], 1e-12)[0])
    f = bfr(O.matmul(h1, p["w1"], p["b1"], epi=O.EPI_GELU_ERF, out_t=O.F64))
    y2 = bfr(O.matmul(f, p["w2"], p["b2"], epi=O.EPI_BIAS, out_t=O.F64) + h1)
    return bfr(O.layernorm(y2, None, p["g2"], p["be2"], 1e-12)[0])


def run_layer(B, S, hd, H, ffn, seed=3):
    bf, f32 = torch.bfloat16, torch.float32
    x, xh = seeded((B * S, hd), "x", seed, dtype=bf)
    dev, host = {}, {}
    for name, shape, lo, hi, dt in [("wqkv", (hd, 3 * hd), -0.05, 0.05, bf),
                                    ("wo", (hd, hd), -0.05, 0.05, bf),
                                    ("w1", (hd, ffn), -0.05, 0.05, bf),
                                    ("w2", (ffn, hd), -0.05, 0.05, bf),
                                    ("bqkv", (3 * hd,), -0.1, 0.1, f32), ("bo", (hd,), -0.1, 0.1, f32),
                                    ("b1", (ffn,), -0.1, 0.1, f32), ("b2", (hd,), -0.1, 0.1, f32),
                                    ("g1", (hd,), 0.9, 1.1, f32), ("be1", (hd,), -0.1, 0.1, f32),
                                    ("g2", (hd,), 0.9, 1.1, f32), ("be2", (hd,), -0.1, 0.1, f32)]:
        dev[name], host[name] = seeded(shape, name, seed, lo, hi, dt)
    y = torch.empty_like(x)
    L = lib()
    ws_bytes = L.afg_encoder_layer_workspace(B, S, hd, ffn, 2)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    d = dev
    afg_check(L.afg_encoder_layer_fwd(
        x.data_ptr(), y.data_ptr(), B, S, hd, H, ffn, d["wqkv"].data_ptr(), d["bqkv"].data_ptr(),
        d["wo"].data_ptr(), d["bo"].data_ptr(), d["g1"].data_ptr(), d["be1"].data_ptr(),
        d["w1"].data_ptr(), d["b1"].data_ptr(), d["w2"].data_ptr(), d["b2"].data_ptr(),
        d["g2"].data_ptr(), d["be2"].data_ptr(), 1e-12, 2, ws.data_ptr(), ws_bytes, st))
    torch.cuda.synchronize()
    return to_host(y), xh, host


def test_bert_layer_full_size_sampled_sequences(cuda):
    """BASELINE configs[4] at full size (B64 x S512, BERT-base): every
    sequence is independent, so sequences 0, 37 and 63 are checked against
    the composed oracle (same tolerance as below)."""
    B, S, hd, H, ffn = 64, 512, 768, 12, 3072
    got, xh, host = run_layer(B, S, hd, H, ffn, seed=4)
    for b in (0, 37, 63):
        sl = slice(b * S, (b + 1) * S)
        want = oracle_bert(xh[sl], host, 1, S, hd, H, ffn)
        check(got[sl], want, 2.0**-5, f"bert layer full size, sequence {b}")
    assert np.isfinite(got).all()


def test_bert_layer_matches_oracle(cuda):
    B, S, hd, H, ffn = 2, 128, 768, 12, 3072
    D = hd // H
    T = B * S
    bf, f32 = torch.bfloat16, torch.float32
    x, xh = seeded((T, hd), "x", 3, dtype=bf)
    wqkv, wqkvh = seeded((hd, 3 * hd), "wqkv", 3, -0.05, 0.05, bf)
    wo, woh = seeded((hd, hd), "wo", 3, -0.05, 0.05, bf)
    w1, w1h = seeded((hd, ffn), "w1", 3, -0.05, 0.05, bf)
    w2, w2h = seeded((ffn, hd), "w2", 3, -0.05, 0.05, bf)
    bqkv, bqkvh = seeded((3 * hd,), "bqkv", 3, -0.1, 0.1, f32)
    bo, boh = seeded((hd,), "bo", 3, -0.1, 0.1, f32)
    b1, b1h = seeded((ffn,), "b1", 3, -0.1, 0.1, f32)
    b2, b2h = seeded((hd,), "b2", 3, -0.1, 0.1, f32)
    g1, g1h = seeded((hd,), "g1", 3, 0.9, 1.1, f32)
    be1, be1h = seeded((hd,), "be1", 3, -0.1, 0.1, f32)
    g2, g2h = seeded((hd,), "g2", 3, 0.9, 1.1, f32)
    be2, be2h = seeded((hd,), "be2", 3, -0.1, 0.1, f32)
    y = torch.empty_like(x)
    L = lib()
    ws_bytes = L.afg_encoder_layer_workspace(B, S, hd, ffn, 2)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    afg_check(L.afg_encoder_layer_fwd(
        x.data_ptr(), y.data_ptr(), B, S, hd, H, ffn, wqkv.data_ptr(), bqkv.data_ptr(),
        wo.data_ptr(), bo.data_ptr(), g1.data_ptr(), be1.data_ptr(), w1.data_ptr(), b1.data_ptr(),
        w2.data_ptr(), b2.data_ptr(), g2.data_ptr(), be2.data_ptr(), 1e-12, 2, ws.data_ptr(),
        ws_bytes, st))
    torch.cuda.synchronize()
    got = to_host(y)

    bfr = lambda a: O.round_to(a, O.BF16)  # noqa: E731
    qkv = bfr(O.matmul(xh, wqkvh, bqkvh, epi=O.EPI_BIAS, out_t=O.F64))
    q = qkv[:, :hd].reshape(B, S, H, D).transpose(0, 2, 1, 3)
    k = qkv[:, hd:2 * hd].reshape(B, S, H, D).transpose(0, 2, 1, 3)
    v = qkv[:, 2 * hd:].reshape(B, S, H, D).transpose(0, 2, 1, 3)
    att = bfr(O.attention(q, k, v, scale=D ** -0.5).transpose(0, 2, 1, 3).reshape(T, hd))
    y1 = bfr(O.matmul(att, woh, boh, epi=O.EPI_BIAS, out_t=O.F64) + xh)
    h1 = bfr(O.layernorm(y1, None, g1h, be1h, 1e-12)[0])
    f = bfr(O.matmul(h1, w1h, b1h, epi=O.EPI_GELU_ERF, out_t=O.F64))
    y2 = bfr(O.matmul(f, w2h, b2h, epi=O.EPI_BIAS, out_t=O.F64) + h1)
    want = bfr(O.layernorm(y2, None, g2h, be2h, 1e-12)[0])
    mr = check(got, want, 2.0**-5, "bert layer")
    assert np.isfinite(got).all()
    print(f"bert layer max_rel {mr:.3e}")


def test_strided_attention_matches_contiguous(cuda):
    from paper_2603_06731_b200 import ops
    B, S, H, D = 2, 256, 4, 64
    qkv, qkvh = seeded((B, S, 3, H, D), "qkv", 9, dtype=torch.bfloat16)
    o = torch.empty((B, S, H, D), dtype=torch.bfloat16, device="cuda")
    qs = (ctypes.c_int64 * 3)(3 * H * D, D, S * 3 * H * D)
    os_ = (ctypes.c_int64 * 3)(H * D, D, S * H * D)
    es = 2
    base = qkv.data_ptr()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    afg_check(lib().afg_attention_fwd_strided(
        base, base + H * D * es, base + 2 * H * D * es, None, o.data_ptr(), B, H, S, S, D, 0.125,
        0, 2, 2, ctypes.cast(qs, ctypes.c_void_p), ctypes.cast(qs, ctypes.c_void_p),
        ctypes.cast(qs, ctypes.c_void_p), ctypes.cast(os_, ctypes.c_void_p), st))
    q = qkvh[:, :, 0].transpose(0, 2, 1, 3)
    k = qkvh[:, :, 1].transpose(0, 2, 1, 3)
    v = qkvh[:, :, 2].transpose(0, 2, 1, 3)
    want = O.attention(q, k, v, scale=0.125).transpose(0, 2, 1, 3)
    check(to_host(o), O.round_to(want, O.BF16), 1e-2, "strided attention")
    # and the contiguous entry point on the same data agrees
    oc = ops.attention(torch.from_numpy(np.ascontiguousarray(q)).to(torch.bfloat16).cuda(),
                       torch.from_numpy(np.ascontiguousarray(k)).to(torch.bfloat16).cuda(),
                       torch.from_numpy(np.ascontiguousarray(v)).to(torch.bfloat16).cuda(),
                       scale=0.125)
    assert torch.equal(oc.transpose(1, 2).contiguous(), o)
