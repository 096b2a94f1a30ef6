"""The drop-in graph executor (afg::gpu::execute via afg_graph_run) on the
BASELINE patterns at 256-512 scale, written in the reference's UNCHANGED graph
API, against the reference interpreter's own outputs
(tests/golden/scale_graphs.*, made by make_scale_golden.py from oracle/_ref).

Every case asserts the plan: the pattern must have run on the tensor-core
kernel it targets (gemm_tc / conv_tc / attn_fwd tcgen05 / gemm_i8 / i8 conv),
or, for the standalone GELU composite, in ONE fused VM launch.

Tolerances (|a-b| <= tol * max(|a|, |b|, 1), interp.cpp:698-730):
  * f32 matmul / conv chains on bf16-valued inputs: 1e-4 (the north-star fp32
    bound): tcgen05 accumulates in fp32 in a different order than the
    interpreter's sequential per-step f32 rounding;
  * f16 attention: 2e-3 (TolProfile::F16Fragment);
  * dequant -> matmul (f32 out): 1e-5 (the integer accumulation is exact, the
    interpreter rounds every partial f32 sum); dequant -> matmul -> quantize:
    at most 1 i8 step (SPEC.md:554 rounding bound), exact on >= 99% of
    elements;
  * the GELU region and the i8 conv: bit-exact (0).
"""
import json
import os

import numpy as np
import pytest

import oracle as O
from paper_2603_06731_b200.graph import execute

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(__file__), "golden")
SPEC = json.load(open(os.path.join(HERE, "scale_graphs.json")))["cases"]
GOLD = np.load(os.path.join(HERE, "scale_graphs.npz"))


def build_inputs(case):
    g = case["graph"]
    inputs = O.random_graph_inputs(g, case["seed"], case["lo"], case["hi"])
    for k in case["bf16"]:
        inputs[k] = O.round_to(inputs[k], O.BF16)
    shapes = {t["id"]: tuple(t["shape"]) for t in g["tensors"]}
    for k, v in case["fixed"].items():
        s = shapes[k]
        if v == "causal":
            m = np.zeros(s)
            iu = np.triu_indices(s[-1], 1)
            m[..., iu[0], iu[1]] = -np.inf
            inputs[k] = m
        elif v == "selector":
            m = np.zeros(s)
            m[..., 0] = 1.0
            inputs[k] = m
        else:
            inputs[k] = np.full(s, v)
    return inputs


@pytest.mark.parametrize("case", SPEC, ids=[c["name"] for c in SPEC])
def test_scale_graph_vs_reference_interpreter(cuda, case):
    out, plan = execute(case["graph"], build_inputs(case), want_plan=True)
    assert any(case["plan"] in p for p in plan), plan
    if case["plan"] == "fused region":
        assert len(plan) == 1, plan  # 14 nests of the reference -> one launch
    for k in case["outputs"]:
        want = GOLD[f"{case['name']}/{k}"].astype(np.float64)
        got = out[k]
        if case["name"].startswith("quant_dequant_matmul_requant"):
            d = np.abs(got - want)
            assert d.max() <= 1.0, f"{k}: max step {d.max()}"
            assert (d == 0).mean() >= 0.99, f"{k}: exact fraction {(d == 0).mean()}"
            continue
        ok, ma, mr, w = O.compare(got, want, case["tol"])
        assert ok, f"{case['name']} {k}: max_rel {mr:.3e} max_abs {ma:.3e} at {w}; plan={plan}"


def test_exact_mode_keeps_f32_bit_exact(cuda):
    """exact=True: the same bf16-valued f32 GEMM+ReLU graph stays on the
    bit-exact fp32 path (SIMT GEMM with the fused epilogue)."""
    case = next(c for c in SPEC if c["name"] == "gemm_bf16_relu_512x256x384")
    out, plan = execute(case["graph"], build_inputs(case), want_plan=True, exact=True)
    assert not any("gemm_tc" in p for p in plan), plan
    want = GOLD[f"{case['name']}/%y"].astype(np.float64)
    assert np.array_equal(out["%y"], want)


def test_quantize_scale_in_double(cuda):
    """quantize(x, scale=0.1) at quotients next to .5: the division runs in
    double like interp.cpp:547-552 (0.35 / 0.1 = 3.4999999999999996 -> 3)."""
    x = np.array([0.35, 0.45, -0.35, 0.25, 1.15, -1.25, 12.65, -12.75] * 8).reshape(8, 8)
    g = {"tensors": [{"id": "x", "shape": [8, 8]}, {"id": "q", "shape": [8, 8], "dtype": "i8"}],
         "ops": [{"op": "quantize", "inputs": ["x"], "output": "q", "attrs": {"scale": 0.1}}]}
    out = execute(g, {"x": x})
    want = np.clip(np.round(np.float32(x).astype(np.float64) / 0.1), -128, 127)
    # np.round is half-to-even; std::round is half-away: build it explicitly
    q = np.float32(x).astype(np.float64) / 0.1
    want = np.clip(np.sign(q) * np.floor(np.abs(q) + 0.5), -128, 127)
    assert np.array_equal(out["%q"], want)
    if O.ref_available():
        assert np.array_equal(out["%q"], O.ref_run(json.dumps(g), {"x": x})["%q"])


def test_int32_values_beyond_2_24_exact(cuda):
    """i8 x i8 -> i32 with |acc| > 2^24: int32 device storage keeps it exact."""
    K = 2048
    a = np.full((4, K), 127.0)
    b = np.full((K, 3), 127.0)
    b[:, 1] = -128.0
    g = {"tensors": [{"id": "a", "shape": [4, K], "dtype": "i8"},
                     {"id": "b", "shape": [K, 3], "dtype": "i8"},
                     {"id": "c", "shape": [4, 3], "dtype": "i32"}],
         "ops": [{"op": "matmul", "inputs": ["a", "b"], "output": "c"}]}
    out = execute(g, {"a": a, "b": b})
    assert out["%c"][0, 0] == 127 * 127 * K and out["%c"][0, 1] == -127 * 128 * K


def test_i8_output_conv_saturates_like_interpreter(cuda):
    """A conv with an i8 output: the interpreter saturates every stored
    partial sum in the loop form and once in the unrolled form
    (frontend.cpp:833-949); the VM conv nest does the same."""
    rng = np.random.default_rng(3)
    for attrs, xs, ws in [({"padding": "same"}, [1, 3, 6, 6], [2, 3, 3, 3]),
                          ({}, [1, 2, 5, 5], [2, 2, 2, 2])]:
        geo = O.conv_geometry(xs[2], xs[3], ws[2], ws[3], (1, 1), (1, 1),
                              attrs.get("padding") == "same")
        g = {"tensors": [{"id": "x", "shape": xs, "dtype": "i8"},
                         {"id": "w", "shape": ws, "dtype": "i8"},
                         {"id": "y", "shape": [1, ws[0], geo[0], geo[1]], "dtype": "i8"}],
             "ops": [{"op": "conv2d", "inputs": ["x", "w"], "output": "y", "attrs": attrs}]}
        x = rng.integers(-100, 100, xs).astype(np.float64)
        w = rng.integers(-9, 9, ws).astype(np.float64)
        out, plan = execute(g, {"x": x, "w": w}, want_plan=True)
        assert np.all(np.abs(out["%y"]) <= 128)
        assert (np.abs(out["%y"]) >= 127).any()  # saturation happened
        if O.ref_available():
            assert np.array_equal(out["%y"], O.ref_run(json.dumps(g), {"x": x, "w": w})["%y"])
