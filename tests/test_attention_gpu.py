"""GPU parity of K3 (fused flash attention on tcgen05) against the oracle
restatement of attentionReference (oracles.cpp:192-227: softmax(QK^T + bias)V
in double), extended with scale and causal masking (== the -inf upper-
triangular additive bias, verified against the reference interpreter in
tests/golden/reference_graphs.json).

Tolerances (reference rule): fp16 inputs 2e-3 (the F16Fragment profile,
interp.cpp:106-118); bf16 inputs 1e-2 (P is rounded to bf16 for
the PV MMA, 2^-8 per term); fp32 SIMT path 1e-5."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2603_06731_b200 import ops
from tests.gpu_util import check, seeded, to_host

pytestmark = pytest.mark.gpu
TOL = {torch.float16: 2e-3, torch.bfloat16: 1e-2, torch.float32: 1e-5}


def attn_case(B, H, N, D, causal=False, dt=torch.float16, scale=1.0, bias=False, Nk=None,
              heads=None, lo=-1.0, hi=1.0, seed=36):
    Nk = Nk or N
    q, qh = seeded((B, H, N, D), "q", seed, lo, hi, dtype=dt)
    k, kh = seeded((B, H, Nk, D), "k", seed, lo, hi, dtype=dt)
    v, vh = seeded((B, H, Nk, D), "v", seed, lo, hi, dtype=dt)
    bb = bbh = None
    if bias:
        bb, bbh = seeded((B, H, N, Nk), "bias", seed, -2.0, 2.0, dtype=torch.float32)
    o = ops.attention(q, k, v, bias=bb, scale=scale, causal=causal, out_dtype=torch.float32)
    got = to_host(o).reshape(B * H, N, D)
    want = O.attention(qh, kh, vh, bias=bbh, scale=scale, causal=causal, heads=heads)
    if heads is None:
        want = want.reshape(B * H, N, D)
    else:
        got = got[heads]
    return check(got, want, TOL[dt], f"attn B{B}H{H}N{N}D{D} causal={causal} {dt}")


@pytest.mark.parametrize("N,D", [(128, 128), (256, 64), (384, 128), (200, 128), (64, 64)])
def test_fp16_noncausal(cuda, N, D):
    attn_case(1, 2, N, D)


@pytest.mark.parametrize("N,D", [(256, 128), (300, 64), (512, 128)])
def test_fp16_causal(cuda, N, D):
    attn_case(2, 2, N, D, causal=True)


def test_scale_and_bias(cuda):
    attn_case(1, 2, 256, 128, scale=128 ** -0.5, bias=True)


def test_bf16_bert_shape(cuda):
    # BERT-base attention: S=512, D=64, scale 1/8
    attn_case(2, 12, 512, 64, dt=torch.bfloat16, scale=0.125)


def test_large_scores_stay_finite(cuda):
    # score entries up to 80 in magnitude
    attn_case(1, 1, 256, 64, lo=-1.6, hi=1.6, scale=1.0)


def test_kv_length_differs(cuda):
    attn_case(1, 2, 128, 128, Nk=320)


def test_full_config_sampled_heads(cuda):
    # BASELINE configs[2]: B8 H16 S2048 D128 fp16, causal, two heads checked
    attn_case(8, 16, 2048, 128, causal=True, heads=np.array([0, 127]))


# D = 128 with several 256-row units per head on the persistent kernel: ragged
# units, ragged keys, bias, bf16 (units cross CTAs' snake walk).
@pytest.mark.parametrize("N,causal,Nk", [(384, False, None), (384, True, None),
                                         (640, True, None), (1024, False, None),
                                         (1024, True, None), (512, False, 700),
                                         (768, True, 900)])
def test_multi_unit_fp16(cuda, N, causal, Nk):
    attn_case(1, 3, N, 128, causal=causal, Nk=Nk, scale=128 ** -0.5)


def test_multi_unit_bias_bf16(cuda):
    attn_case(1, 2, 512, 128, bias=True, scale=128 ** -0.5)
    attn_case(2, 2, 768, 128, causal=True, dt=torch.bfloat16, scale=128 ** -0.5)


def test_full_config_noncausal_sampled_heads(cuda):
    attn_case(8, 16, 2048, 128, heads=np.array([3, 64, 126]), scale=128 ** -0.5)


def test_simt_path_reference_shapes(cuda):
    # the reference test's attention graph shape [1,2,8,4] (test_frontend.cpp:275-305)
    attn_case(1, 2, 8, 4, dt=torch.float32, bias=True)
    attn_case(2, 1, 7, 16, dt=torch.float32, causal=True)
    attn_case(1, 1, 1, 4, dt=torch.float32)  # N = 1: output = V row


def test_concurrent_streams_dynamic_queue(cuda):
    # the dynamic unit queue keeps one counter pair per stream: two attention
    # launches running concurrently on two streams must each produce the same
    # result as alone (bit-identical: a unit's arithmetic does not depend on
    # which CTA takes it)
    outs = []
    ins = []
    for seed in (41, 42):
        q, _ = seeded((4, 8, 1024, 128), "q", seed, dtype=torch.float16)
        k, _ = seeded((4, 8, 1024, 128), "k", seed, dtype=torch.float16)
        v, _ = seeded((4, 8, 1024, 128), "v", seed, dtype=torch.float16)
        ins.append((q, k, v))
        outs.append(ops.attention(q, k, v, scale=128 ** -0.5, causal=True))
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for _ in range(5):
        got = []
        for s, (q, k, v) in zip(streams, ins):
            with torch.cuda.stream(s):
                got.append(ops.attention(q, k, v, scale=128 ** -0.5, causal=True))
        torch.cuda.synchronize()
        for g, w in zip(got, outs):
            assert torch.equal(g, w)
