"""GPU parity of K2 (implicit-GEMM NHWC convolution with fused bias+ReLU on
tcgen05, im2col TMA) and of the direct NCHW kernel that carries the
reference's own conv2d semantics (stride / dilation / same / transposed,
frontend.cpp:752-970; convReference oracles.cpp:78-120).

Tolerances: bf16 output one bf16 ulp (2^-7) against the oracle rounded to
bf16 on the same rounded inputs; fp32 paths 1e-5."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2603_06731_b200 import Epilogue, ops
from tests.gpu_util import check, seeded, to_host

pytestmark = pytest.mark.gpu

EPI = {Epilogue.NONE: O.EPI_NONE, Epilogue.BIAS: O.EPI_BIAS, Epilogue.BIAS_RELU: O.EPI_RELU}


def conv_case(B, H, W, C, OC, k, stride, pad, dt=torch.bfloat16, epi=Epilogue.BIAS_RELU,
              dil=1, seed=44, images=None):
    x, xh = seeded((B, H, W, C), "x", seed, dtype=dt)
    w, wh = seeded((OC, k, k, C), "w", seed, -0.2, 0.2, dtype=dt)
    bias, bh = seeded((OC,), "bias", seed, dtype=torch.float32)
    y = ops.conv2d_nhwc(x, w, bias if epi != Epilogue.NONE else None, (stride, stride),
                        (pad, pad), (dil, dil), epilogue=epi)
    got = to_host(y)
    code = {torch.bfloat16: O.BF16, torch.float16: O.F16, torch.float32: O.F32}[dt]
    want = O.conv_nhwc(xh, wh, bh, (stride, stride), (pad, pad), (dil, dil), epi=EPI[epi],
                       out_t=O.F64, images=images)
    want = O.round_to(want, code)
    if images is not None:
        got = got[images]
    tol = {torch.bfloat16: 2.0**-7, torch.float16: 2.0**-10, torch.float32: 1e-5}[dt]
    return check(got, want, tol, f"conv {B}x{H}x{W}x{C}->{OC} k{k} s{stride} p{pad}")


@pytest.mark.parametrize("B,H,W,C,OC,k,s,p", [
    (2, 8, 8, 64, 64, 3, 1, 1),     # 3x3 same
    (2, 14, 14, 128, 128, 3, 2, 1),  # 3x3 stride 2, even input (PyTorch pad=1)
    (1, 7, 7, 64, 256, 3, 1, 1),    # 7x7 tiles crossing images
    (3, 9, 11, 64, 96, 3, 1, 0),    # odd extents, valid, ragged OC
    (2, 8, 8, 64, 256, 1, 1, 0),    # 1x1: plain GEMM path
    (2, 14, 14, 128, 64, 1, 2, 0),  # 1x1 stride-2 downsample
])
def test_implicit_gemm_tc(cuda, B, H, W, C, OC, k, s, p):
    conv_case(B, H, W, C, OC, k, s, p)


# 3x3 / stride 1 / pad 1 with 20 <= W <= 62 runs the halo-tiled kernel (input
# staged once per tile and channel chunk, taps as shifted smem windows): both
# halo pitches (P = 32 / 64), rows past the image bottom (H % R != 0), ragged
# OC, several channel chunks, fp16, no epilogue; narrower images (the im2col
# path) alongside.
@pytest.mark.parametrize("B,H,W,C,OC,dt,epi", [
    (2, 56, 56, 64, 64, torch.bfloat16, Epilogue.BIAS_RELU),
    (2, 28, 28, 128, 128, torch.bfloat16, Epilogue.BIAS_RELU),
    (2, 14, 14, 256, 256, torch.bfloat16, Epilogue.BIAS_RELU),
    (3, 23, 21, 64, 96, torch.float16, Epilogue.BIAS),
    (1, 31, 62, 192, 64, torch.bfloat16, Epilogue.NONE),
    (2, 57, 40, 128, 320, torch.bfloat16, Epilogue.BIAS_RELU),
])
def test_halo_conv_3x3(cuda, B, H, W, C, OC, dt, epi):
    conv_case(B, H, W, C, OC, 3, 1, 1, dt=dt, epi=epi)


# im2col convs with OC >= 256 and K >= 768 on CTA-pair 256 x 256 tiles (both
# CTAs gather their own 128 output pixels); sampled images at full batch.
@pytest.mark.parametrize("B,H,C,OC,s", [(128, 14, 256, 256, 1), (64, 28, 256, 512, 2)])
def test_im2col_pair_tiles(cuda, B, H, C, OC, s):
    conv_case(B, H, H, C, OC, 3, s, 1, images=np.array([0, B // 2 + 1, B - 1]))


def test_implicit_gemm_dilation_and_no_epilogue(cuda):
    conv_case(2, 12, 12, 64, 64, 3, 1, 2, dil=2, epi=Epilogue.NONE)


def test_resnet_layer_full_batch_sampled_images(cuda):
    # ResNet-50 layer2 3x3 128->128 at 28x28, batch 32 (one B200's shard of 256)
    conv_case(32, 28, 28, 128, 128, 3, 1, 1, images=np.array([0, 17, 31]))


def test_direct_nhwc_fallback_small_channels(cuda):
    conv_case(2, 9, 9, 3, 8, 3, 2, 1, dt=torch.float32)
    conv_case(1, 6, 6, 20, 12, 3, 1, 1, dt=torch.bfloat16)


def test_pack_filter(cuda):
    w, wh = seeded((8, 5, 3, 3), "w", 1, dtype=torch.float32)
    p = ops.conv_pack_filter(w)
    assert np.array_equal(to_host(p), wh.transpose(0, 2, 3, 1))


@pytest.mark.parametrize("attrs,ins,ws", [
    ({}, (2, 3, 9, 8), (4, 3, 3, 3)),
    ({"stride": 2}, (1, 2, 9, 9), (3, 2, 3, 3)),
    ({"dilation": 2}, (1, 2, 9, 9), (3, 2, 3, 3)),
    ({"padding": "same"}, (1, 2, 8, 8), (3, 2, 3, 3)),
    ({"padding": "same", "stride": 2}, (1, 2, 9, 9), (3, 2, 3, 3)),
    ({"padding": "same", "stride": 2}, (1, 2, 8, 8), (3, 2, 3, 3)),  # pad_begin 0 (§0.7)
    ({"transposed": True, "stride": 2}, (1, 2, 4, 4), (2, 3, 2, 2)),
    ({"transposed": True, "stride": 2, "padding": "same"}, (1, 2, 4, 4), (2, 3, 3, 3)),
])
def test_direct_nchw_reference_semantics(cuda, attrs, ins, ws):
    s = attrs.get("stride", 1)
    d = attrs.get("dilation", 1)
    tr = attrs.get("transposed", False)
    x, xh = seeded(ins, "in", 21, 0.0, 1.0, dtype=torch.float32)
    w, wh = seeded(ws, "w", 21, 0.0, 1.0, dtype=torch.float32)
    oh, ow, py, px = O.conv_geometry(ins[2], ins[3], ws[2], ws[3], (s, s), (d, d),
                                     attrs.get("padding") == "same", tr)
    y = ops.conv2d_nchw(x, w, (s, s), (d, d), (py, px), tr, (oh, ow))
    want = O.conv_nchw(xh, wh, (s, s), (d, d), (py, px), tr, (oh, ow))
    check(to_host(y), want, 1e-6, f"conv nchw {attrs}")
