"""The SPEC's edge-case grids on the tensor-core paths (the
reference modules are stubs).

Conv: stride {1,2} x dilation {1,2} x padding
{valid, same} x transposed {no, yes} x odd / even extents = 32 configs, as
reference-API conv2d graphs (NCHW / OIHW, IOHW transposed) with bf16-valued f32
tensors, which the executor must run on the implicit-GEMM tcgen05 kernel
(plan: conv_tc). Checked against the direct-conv restatement of
convReference (oracles.cpp:78-120, pinned by tests/test_oracle.py) on the
same inputs: 1e-4 (fp32 accumulation order). Zero-pad neutrality: the same
conv with the channels zero-padded from 64 to 128 is bit-identical.

Attention: B, H in {1, 2}, N in {1, 7, 8, 64}
(+ ragged 200), f16: D in {64, 128} on the tcgen05 kernel (causal and not),
D in {4, 16} on the SIMT kernel; 2e-3 (F16Fragment) vs attentionReference;
N = 1 gives the V row; scores of magnitude up to 80 stay finite."""
import itertools

import numpy as np
import pytest
import torch

import oracle as O
from paper_2603_06731_b200 import ops
from paper_2603_06731_b200.graph import execute
from tests.gpu_util import to_host

pytestmark = pytest.mark.gpu

CONV_GRID = list(itertools.product([1, 2], [1, 2], ["valid", "same"], [False, True], [8, 9]))


def conv_case(stride, dil, padding, transposed, hw, C=64, OC=64, pad_channels=0):
    x = O.round_to(O.random_tensor((1, C, hw, hw), "%x", 70 + hw, -1, 1), O.BF16)
    wshape = (C, OC, 3, 3) if transposed else (OC, C, 3, 3)
    w = O.round_to(O.random_tensor(wshape, "%w", 71, -0.2, 0.2), O.BF16)
    geo = O.conv_geometry(hw, hw, 3, 3, (stride, stride), (dil, dil), padding == "same",
                          transposed)
    OH, OW, py, px = geo
    if pad_channels:
        x = np.concatenate([x, np.zeros((1, pad_channels, hw, hw))], axis=1)
        w = np.concatenate([w, np.zeros((pad_channels,) + wshape[1:])], axis=0) if transposed \
            else np.concatenate([w, np.zeros((OC, pad_channels, 3, 3))], axis=1)
    Cx = x.shape[1]
    g = {"tensors": [{"id": "x", "shape": [1, Cx, hw, hw]}, {"id": "w", "shape": list(w.shape)},
                     {"id": "y", "shape": [1, OC, OH, OW]}],
         "ops": [{"op": "conv2d", "inputs": ["x", "w"], "output": "y",
                  "attrs": {"stride": stride, "dilation": dil, "padding": padding,
                            "transposed": transposed}}]}
    return g, x, w, (OH, OW, py, px)


@pytest.mark.parametrize("stride,dil,padding,transposed,hw", CONV_GRID,
                         ids=[f"s{s}d{d}{p}{'T' if t else ''}{h}" for s, d, p, t, h in CONV_GRID])
def test_conv_grid_on_tensor_cores(cuda, stride, dil, padding, transposed, hw):
    g, x, w, (OH, OW, py, px) = conv_case(stride, dil, padding, transposed, hw)
    out, plan = execute(g, {"x": x, "w": w}, want_plan=True)
    assert any("conv_tc" in p for p in plan), plan
    want = O.conv_nchw(x, w, (stride, stride), (dil, dil), (py, px), transposed, (OH, OW),
                       out_t=O.F64)
    ok, ma, mr, wi = O.compare(out["%y"], want, 1e-4)
    assert ok, f"max_rel {mr:.3e} at {wi}; plan={plan}"


@pytest.mark.parametrize("transposed", [False, True])
def test_conv_zero_pad_neutrality(cuda, transposed):
    g64, x64, w64, _ = conv_case(2, 1, "same", transposed, 9)
    g128, x128, w128, _ = conv_case(2, 1, "same", transposed, 9, pad_channels=64)
    a = execute(g64, {"x": x64, "w": w64})["%y"]
    b = execute(g128, {"x": x128, "w": w128})["%y"]
    assert np.array_equal(a, b)


ATTN_GRID = list(itertools.product([1, 2], [1, 2], [1, 7, 8, 64, 200], [64, 128], [False, True]))


@pytest.mark.parametrize("B,H,N,D,causal", ATTN_GRID,
                         ids=[f"B{b}H{h}N{n}D{d}{'c' if c else ''}" for b, h, n, d, c in ATTN_GRID])
def test_attention_grid_f16_tensor_cores(cuda, B, H, N, D, causal):
    q, k, v = (O.round_to(O.random_tensor((B, H, N, D), "%" + t, 80 + N, -1, 1), O.F16)
               for t in "qkv")
    tq, tk, tv = (torch.from_numpy(a).half().cuda() for a in (q, k, v))
    o = ops.attention(tq, tk, tv, scale=D ** -0.5, causal=causal, out_dtype=torch.float32)
    want = O.attention(q, k, v, scale=D ** -0.5, causal=causal)
    ok, ma, mr, w = O.compare(to_host(o), want, 2e-3)
    assert ok, f"max_rel {mr:.3e} at {w}"
    if N == 1:  # one key -> the output is the V row
        assert np.allclose(to_host(o), v, rtol=0, atol=1e-3)


@pytest.mark.parametrize("B,H,N,D", list(itertools.product([1, 2], [1, 2], [1, 7, 8, 64],
                                                             [4, 16])))
def test_attention_grid_f16_small_head_dim(cuda, B, H, N, D):
    q, k, v = (O.round_to(O.random_tensor((B, H, N, D), "%" + t, 90 + N, -1, 1), O.F16)
               for t in "qkv")
    tq, tk, tv = (torch.from_numpy(a).half().cuda() for a in (q, k, v))
    o = ops.attention(tq, tk, tv, scale=1.0, causal=False, out_dtype=torch.float32)
    ok, ma, mr, w = O.compare(to_host(o), O.attention(q, k, v), 2e-3)
    assert ok, f"max_rel {mr:.3e} at {w}"


@pytest.mark.parametrize("D", [64, 128])
def test_attention_large_scores_stay_finite(cuda, D):
    """scores up to 80 in magnitude: finite outputs."""
    N = 256
    rng = np.random.default_rng(1)
    q = np.full((1, 1, N, D), 1.0)
    k = O.round_to(rng.choice([-1.0, 1.0], (1, 1, N, D)), O.F16)
    v = O.round_to(rng.uniform(-1, 1, (1, 1, N, D)), O.F16)
    scale = 80.0 / D  # |q.k| * scale reaches 80
    tq, tk, tv = (torch.from_numpy(a).half().cuda() for a in (q, k, v))
    o = to_host(ops.attention(tq, tk, tv, scale=scale, out_dtype=torch.float32))
    assert np.isfinite(o).all()
    ok, ma, mr, w = O.compare(o, O.attention(q, k, v, scale=scale), 2e-3)
    assert ok, mr
