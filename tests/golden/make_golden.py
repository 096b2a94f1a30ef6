"""Regenerates tests/golden/reference_graphs.json from the UNMODIFIED reference
(oracle/_ref/libafref.so, built from /root/reference/proj by oracle/Makefile).

For every graph below it records the inputs the reference's own generator
makes (af::makeRandomInputs, interp.cpp:846-853, as checkLowering does,
test_frontend.cpp:22-37), the outputs of af::interpret on the lowered program
and of oracle::evalGraphReference. The first group are the graphs of the
reference's test_frontend.cpp (same shapes, same seeds); the second group are
the BASELINE-config patterns expressed in the unchanged graph API
 at small sizes: matmul+bias+ReLU, matmul+bias+GELU
(14-nest composite), attention with and without a causal -inf bias, softmax,
NHWC conv via transposes, pre-padded stride-2 conv.

Run here (needs the reference build):  python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import oracle as O  # noqa: E402
from oracle.graphs import (T, attention_graph, conv_graph, matmul_epi_graph,  # noqa: E402
                           nhwc_conv_graph)

OUT = os.path.join(os.path.dirname(__file__), "reference_graphs.json")


# ---- graphs of test_frontend.cpp (shapes + seeds verbatim) ----------------
FRONTEND = [
    ("matmul_4x4", 11, {"tensors": [T("a", [4, 4]), T("b", [4, 4]), T("c", [4, 4])],
                        "ops": [{"op": "matmul", "inputs": ["a", "b"], "output": "c"}]}),
    ("softmax_2x3", 12, {"tensors": [T("x", [2, 3]), T("y", [2, 3])],
                         "ops": [{"op": "softmax", "inputs": ["x"], "output": "y",
                                  "attrs": {"axis": -1}}]}),
    ("blur_chain", 13, {"tensors": [T("img", [3, 1, 34, 30]), T("wx", [1, 1, 1, 3]),
                                    T("wy", [1, 1, 3, 1]), T("bx", [3, 1, 34, 28]),
                                    T("by", [3, 1, 32, 28])],
                        "ops": [{"op": "conv2d", "inputs": ["img", "wx"], "output": "bx"},
                                {"op": "conv2d", "inputs": ["bx", "wy"], "output": "by"}]}),
    ("conv_direct", 14, conv_graph({}, [2, 3, 9, 8], [4, 3, 3, 3], [2, 4, 7, 6])),
    ("conv_stride2", 21, conv_graph({"stride": 2}, [1, 2, 9, 9], [3, 2, 3, 3], [1, 3, 4, 4])),
    ("conv_dil2", 22, conv_graph({"dilation": 2}, [1, 2, 9, 9], [3, 2, 3, 3], [1, 3, 5, 5])),
    ("conv_same", 23, conv_graph({"padding": "same"}, [1, 2, 8, 8], [3, 2, 3, 3], [1, 3, 8, 8])),
    ("conv_same_s2", 24, conv_graph({"padding": "same", "stride": 2}, [1, 2, 9, 9],
                                    [3, 2, 3, 3], [1, 3, 5, 5])),
    ("conv_transposed_s2", 25, conv_graph({"transposed": True, "stride": 2}, [1, 2, 4, 4],
                                          [2, 3, 2, 2], [1, 3, 8, 8])),
    ("conv_transposed_same", 26, conv_graph({"transposed": True, "stride": 2, "padding": "same"},
                                            [1, 2, 4, 4], [2, 3, 3, 3], [1, 3, 8, 8])),
    ("misc_ops", 31, {"tensors": [T("a", [3, 5]), T("b", [3, 5]), T("c", [3, 5]), T("d", [3, 5]),
                                  T("e", [5, 3]), T("f", [3]), T("g", [3, 5])],
                      "ops": [{"op": "add", "inputs": ["a", "b"], "output": "c"},
                              {"op": "mul", "inputs": ["c", "a"], "output": "d"},
                              {"op": "transpose", "inputs": ["d", "d"], "output": "e",
                               "attrs": {"perm": [1, 0]}},
                              {"op": "reduce", "inputs": ["d"], "output": "f",
                               "attrs": {"op": "max", "axis": 1}},
                              {"op": "broadcast_in_dim", "inputs": ["f"], "output": "g",
                               "attrs": {"dims": [0]}}]}),
    ("batch_matmul", 32, {"tensors": [T("x", [2, 2, 3, 4]), T("y", [2, 2, 4, 5]),
                                      T("z", [2, 2, 3, 5])],
                          "ops": [{"op": "batch_matmul", "inputs": ["x", "y"], "output": "z"}]}),
    ("reshape_exp", 33, {"tensors": [T("x", [3, 1, 4]), T("y", [12]), T("z", [2, 6]),
                                     T("w", [2, 6])],
                         "ops": [{"op": "reshape", "inputs": ["x"], "output": "y"},
                                 {"op": "reshape", "inputs": ["y"], "output": "z"},
                                 {"op": "exp", "inputs": ["z"], "output": "w"}]}),
    ("quant_dequant", 34, {"tensors": [T("x", [4, 6]), T("q", [4, 6], "i8"), T("y", [4, 6])],
                           "ops": [{"op": "quantize", "inputs": ["x"], "output": "q",
                                    "attrs": {"scale": 0.03125}},
                                   {"op": "dequantize", "inputs": ["q"], "output": "y",
                                    "attrs": {"scale": 0.03125}}]}),
    ("sub_max", 35, {"tensors": [T("a", [4, 4]), T("b", [4, 4]), T("c", [4, 4]), T("d", [4, 4])],
                     "ops": [{"op": "sub", "inputs": ["a", "b"], "output": "c"},
                             {"op": "max", "inputs": ["c", "b"], "output": "d"}]}),
    ("attention_1x2x8x4", 36, {"tensors": [T("q", [1, 2, 8, 4]), T("k", [1, 2, 8, 4]),
                                           T("kt", [1, 2, 4, 8]), T("v", [1, 2, 8, 4]),
                                           T("bias", [1, 2, 8, 8]), T("qk", [1, 2, 8, 8]),
                                           T("qkb", [1, 2, 8, 8]), T("soft", [1, 2, 8, 8]),
                                           T("out", [1, 2, 8, 4])],
                               "ops": [{"op": "transpose", "inputs": ["k"], "output": "kt",
                                        "attrs": {"perm": [0, 1, 3, 2]}},
                                       {"op": "batch_matmul", "inputs": ["q", "kt"],
                                        "output": "qk"},
                                       {"op": "add", "inputs": ["qk", "bias"], "output": "qkb"},
                                       {"op": "softmax", "inputs": ["qkb"], "output": "soft",
                                        "attrs": {"axis": -1}},
                                       {"op": "batch_matmul", "inputs": ["soft", "v"],
                                        "output": "out"}]}),
]


PATTERNS = []
for name, (M, N, K), act in [("mm_bias_relu_48x40x24", (48, 40, 24), "relu"),
                             ("mm_bias_gelu_32x24x16", (32, 24, 16), "gelu"),
                             ("mm_bias_16x64x32", (16, 64, 32), None)]:
    g, fixed = matmul_epi_graph(M, N, K, act)
    PATTERNS.append((name, 41, g, fixed, -1.0, 1.0))
for name, causal in [("attn_f16_1x2x16x8", False), ("attn_f16_causal_1x2x16x8", True)]:
    g, fixed = attention_graph(1, 2, 16, 8, causal)
    PATTERNS.append((name, 42, g, fixed, -1.0, 1.0))
PATTERNS.append(("softmax_f16in_4x64", 43,
                 {"tensors": [T("x", [4, 64], "f16"), T("y", [4, 64])],
                  "ops": [{"op": "softmax", "inputs": ["x"], "output": "y",
                           "attrs": {"axis": -1}}]}, {}, -4.0, 4.0))
g, fixed = nhwc_conv_graph(2, 6, 6, 4, 8, 3, 1, "same")
PATTERNS.append(("nhwc_conv3x3_same_relu", 44, g, fixed, -1.0, 1.0))
g, fixed = nhwc_conv_graph(1, 10, 10, 4, 8, 3, 2, "valid")  # pre-padded 8x8, pad=1
PATTERNS.append(("nhwc_conv3x3_s2_prepadded_relu", 45, g, fixed, -1.0, 1.0))


def enc(a):
    a = np.asarray(a, dtype=np.float64)
    return {"shape": list(a.shape),
            "data": [None if not np.isfinite(v) else float(v) for v in a.ravel()],
            "nonfinite": {str(i): ("inf" if v > 0 else "-inf") for i, v in enumerate(a.ravel())
                          if not np.isfinite(v)}}


FIXED = {}


def main():
    cases = []
    for name, seed, g in FRONTEND:
        gj = json.dumps(g)
        inputs = {k[1:]: v for k, v in O.ref_random_inputs(gj, seed).items()}
        interp = O.ref_run(gj, inputs, "interpret")
        orc = O.ref_run(gj, inputs, "oracle")
        cases.append({"name": name, "group": "test_frontend", "seed": seed, "lo": 0.0, "hi": 1.0,
                      "graph": g, "inputs": {k: enc(v) for k, v in inputs.items()},
                      "interpret": {k: enc(v) for k, v in interp.items()},
                      "oracle": {k: enc(v) for k, v in orc.items()}})
    for name, seed, g, fixed, lo, hi in PATTERNS:
        FIXED[name] = fixed
        gj = json.dumps(g)
        inputs = {k[1:]: v for k, v in O.ref_random_inputs(gj, seed, lo, hi).items()}
        inputs.update(fixed)
        interp = O.ref_run(gj, inputs, "interpret")
        orc = O.ref_run(gj, inputs, "oracle")
        cases.append({"name": name, "group": "baseline_pattern", "seed": seed, "lo": lo, "hi": hi,
                      "fixed": sorted(fixed), "graph": g,
                      "inputs": {k: enc(v) for k, v in inputs.items()},
                      "interpret": {k: enc(v) for k, v in interp.items()},
                      "oracle": {k: enc(v) for k, v in orc.items()}})
    # the reference-side driver spec (integration/check_lowering_gpu.cpp)
    spec = []
    for c in cases:
        entry = {"name": c["name"], "graph": c["graph"], "seed": c["seed"], "lo": c["lo"],
                 "hi": c["hi"],
                 "profile": "Int" if c["name"] == "quant_dequant" else
                 ("F16Fragment" if "f16" in c["name"] else "F32")}
        if c.get("fixed"):
            entry["fixed"] = {k: [("-inf" if v == -np.inf else "inf") if not np.isfinite(v) else v
                                  for v in np.asarray(FIXED[c["name"]][k]).ravel().tolist()]
                              for k in c["fixed"]}
        spec.append(entry)
    with open(os.path.join(os.path.dirname(__file__), "check_lowering_cases.json"), "w") as f:
        json.dump({"cases": spec}, f, separators=(",", ":"))
    with open(OUT, "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py",
                   "reference": "/root/reference/proj (AffineForge), built by oracle/Makefile",
                   "cases": cases}, f, separators=(",", ":"))
    print(f"wrote {OUT}: {len(cases)} cases, {os.path.getsize(OUT) / 1024:.0f} KiB")


if __name__ == "__main__":
    main()
