"""Regenerates tests/golden/scale_graphs.{json,npz}: the BASELINE patterns at
256-512 scale, written in the reference's unchanged graph API (SURVEY.md App.
B), with the outputs of the UNMODIFIED reference interpreter (oracle/_ref:
lowerGraphToAffine + af::interpret) on them.

Inputs are the reference generator's (af::makeRandomInputs, interp.cpp:846-853)
with the listed tensors then rounded to bf16 (RNE) -- the App. B convention for
bf16 data carried in f32 tensors -- and the constant tensors (zeros, GELU
coefficients, selector mask, causal mask, uniform scale) overwritten. The
tests (tests/test_graph_scale_gpu.py) regenerate the inputs with the pinned
restatement (oracle.random_graph_inputs) and compare against the stored
outputs (float32: every value is an f32 / f16 / integer the interpreter
stored, so the fixture is lossless).

Run here (needs the reference build, ~2 min on 8 cores):
    python tests/golden/make_scale_golden.py
"""
from __future__ import annotations

import json
import math
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import oracle as O  # noqa: E402
from oracle.graphs import T, matmul_epi_graph, nhwc_conv_graph  # noqa: E402

HERE = os.path.dirname(__file__)


def attention_graph_scaled(B, H, N, D, causal, scale, dtype="f16"):
    """transpose -> batch_matmul -> mul(scale) -> [add(causal -inf)] ->
    softmax -> batch_matmul (test_frontend.cpp:275-305 + App. B scale)."""
    g = {"tensors": [T("q", [B, H, N, D], dtype), T("k", [B, H, N, D], dtype),
                     T("kt", [B, H, D, N], dtype), T("v", [B, H, N, D], dtype),
                     T("qk", [B, H, N, N]), T("sc", [B, H, N, N]), T("qs", [B, H, N, N]),
                     T("soft", [B, H, N, N]), T("out", [B, H, N, D])],
         "ops": [{"op": "transpose", "inputs": ["k"], "output": "kt",
                  "attrs": {"perm": [0, 1, 3, 2]}},
                 {"op": "batch_matmul", "inputs": ["q", "kt"], "output": "qk"},
                 {"op": "mul", "inputs": ["qk", "sc"], "output": "qs"}]}
    fixed = {"sc": np.full((B, H, N, N), float(np.float32(scale)))}
    src = "qs"
    if causal:
        g["tensors"] += [T("mask", [B, H, N, N]), T("qkb", [B, H, N, N])]
        g["ops"].append({"op": "add", "inputs": ["qs", "mask"], "output": "qkb"})
        m = np.zeros((B, H, N, N))
        iu = np.triu_indices(N, 1)
        m[..., iu[0], iu[1]] = -np.inf
        fixed["mask"] = m
        src = "qkb"
    g["ops"] += [{"op": "softmax", "inputs": [src], "output": "soft", "attrs": {"axis": -1}},
                 {"op": "batch_matmul", "inputs": ["soft", "v"], "output": "out"}]
    return g, fixed


def gelu_only_graph(M, N):
    """The 14-nest tanh-GELU composite alone (no matmul in front): the fused
    VM region must run it in one launch."""
    g, fixed = matmul_epi_graph(M, N, 8, "gelu")
    # drop matmul/bias: x = cb becomes an input
    g["ops"] = [o for o in g["ops"] if o["output"] not in ("c", "bb", "cb")]
    g["tensors"] = [t for t in g["tensors"] if t["id"] not in ("a", "b", "bias", "c", "bb")]
    return g, fixed


def quant_graph(M, N, K, requant=True):
    """dequantize(qa) . dequantize(qb) [-> quantize]."""
    g = {"tensors": [T("qa", [M, K], "i8"), T("qb", [K, N], "i8"), T("a", [M, K]),
                     T("b", [K, N]), T("c", [M, N])],
         "ops": [{"op": "dequantize", "inputs": ["qa"], "output": "a", "attrs": {"scale": 0.05}},
                 {"op": "dequantize", "inputs": ["qb"], "output": "b", "attrs": {"scale": 0.03}},
                 {"op": "matmul", "inputs": ["a", "b"], "output": "c"}]}
    if requant:
        g["tensors"].append(T("q", [M, N], "i8"))
        g["ops"].append({"op": "quantize", "inputs": ["c"], "output": "q",
                         "attrs": {"scale": 0.07}})
    return g, {}


def conv_i8_graph(B, C, H, W, OC, k, padding):
    geo = O.conv_geometry(H, W, k, k, (1, 1), (1, 1), padding == "same")
    g = {"tensors": [T("x", [B, C, H, W], "i8"), T("w", [OC, C, k, k], "i8"),
                     T("y", [B, OC, geo[0], geo[1]], "i32")],
         "ops": [{"op": "conv2d", "inputs": ["x", "w"], "output": "y",
                  "attrs": {"padding": padding}}]}
    return g, {}


# name, seed, graph builder, lo, hi, tensors rounded to bf16, tolerance, plan marker
def cases():
    out = []
    g, f = matmul_epi_graph(256, 256, 256, "gelu")
    out.append(("gemm_bf16_gelu_256", 51, g, f, -1.0, 1.0, ["a", "b"], 1e-4, "gemm_tc bf16"))
    g, f = matmul_epi_graph(512, 256, 384, "relu")
    out.append(("gemm_bf16_relu_512x256x384", 52, g, f, -1.0, 1.0, ["a", "b"], 1e-4,
                "gemm_tc bf16"))
    g, f = nhwc_conv_graph(2, 16, 16, 64, 128, 3, 1, "same")
    out.append(("nhwc_conv3x3_same_16x16_64to128", 53, g, f, -1.0, 1.0, ["x", "w"], 1e-4,
                "conv_tc"))
    g, f = nhwc_conv_graph(1, 32, 32, 64, 64, 3, 1, "same")
    out.append(("nhwc_conv3x3_same_32x32_halo", 54, g, f, -1.0, 1.0, ["x", "w"], 1e-4,
                "conv_tc"))
    g, f = nhwc_conv_graph(2, 34, 34, 64, 64, 3, 2, "valid")  # pre-padded 32x32, pad 1
    out.append(("nhwc_conv3x3_s2_prepadded_34", 55, g, f, -1.0, 1.0, ["x", "w"], 1e-4,
                "conv_tc"))
    g, f = attention_graph_scaled(1, 2, 256, 128, True, 128 ** -0.5)
    out.append(("attn_f16_causal_scale_d128_n256", 56, g, f, -1.0, 1.0, [], 2e-3,
                "attn_fwd tcgen05"))
    g, f = attention_graph_scaled(1, 2, 256, 64, False, 0.125)
    out.append(("attn_f16_scale_d64_n256", 57, g, f, -1.0, 1.0, [], 2e-3, "attn_fwd tcgen05"))
    g, f = gelu_only_graph(64, 96)
    out.append(("gelu_composite_region_64x96", 58, g, f, -3.0, 3.0, [], 0.0, "fused region"))
    g, f = quant_graph(128, 128, 128)
    out.append(("quant_dequant_matmul_requant_128", 59, g, f, 0.0, 1.0, [], 1.0, "afg_gemm_i8"))
    g, f = quant_graph(128, 96, 160, requant=False)
    out.append(("quant_dequant_matmul_f32_128x96x160", 60, g, f, 0.0, 1.0, [], 1e-5,
                "afg_gemm_i8"))
    g, f = conv_i8_graph(2, 32, 10, 10, 48, 3, "same")
    out.append(("conv_i8_same_32to48", 61, g, f, 0.0, 1.0, [], 0.0, "afg_conv2d_nhwc_i8"))
    from oracle.graphs import bert_layer_graph
    g, f, _ = bert_layer_graph(64, 128, 2, 512)
    out.append(("bert_layer_graph_s64_h128", 62, g, f, -0.5, 0.5,
                ["x", "wq", "wk", "wv", "wo", "w1", "w2"], 1e-4, "afg_attention_fwd"))
    return out


def run_case(c):
    name, seed, g, fixed, lo, hi, bf16, tol, marker = c
    gj = json.dumps(g)
    inputs = {k[1:]: v for k, v in O.ref_random_inputs(gj, seed, lo, hi).items()}
    for k in bf16:
        inputs[k] = O.round_to(inputs[k], O.BF16)
    inputs.update(fixed)
    out = O.ref_run(gj, inputs, "interpret")
    return name, {k: np.asarray(v, dtype=np.float32) for k, v in out.items()}


def main():
    cs = cases()
    with ProcessPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = dict(ex.map(run_case, cs))
    arrays = {}
    spec = []
    for name, seed, g, fixed, lo, hi, bf16, tol, marker in cs:
        for k, v in results[name].items():
            arrays[f"{name}/{k}"] = v
        spec.append({"name": name, "seed": seed, "graph": g, "lo": lo, "hi": hi, "bf16": bf16,
                     "fixed": {k: ("causal" if k == "mask" and "attn" in name else
                                   float(np.asarray(v).ravel()[0]) if np.all(np.asarray(v) ==
                                                                          np.asarray(v).ravel()[0])
                                   else "selector")
                               for k, v in fixed.items()},
                     "tol": tol, "plan": marker, "outputs": sorted(results[name])})
    np.savez_compressed(os.path.join(HERE, "scale_graphs.npz"), **arrays)
    with open(os.path.join(HERE, "scale_graphs.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_scale_golden.py", "cases": spec}, f, indent=1)
    print("wrote", len(spec), "cases")


if __name__ == "__main__":
    main()
