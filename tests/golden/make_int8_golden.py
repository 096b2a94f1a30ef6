"""Generates tests/golden/int8_matmul.json: i8 x i8 -> i32 matmul graphs run
through the UNMODIFIED reference (oracle/_ref: lowerGraphToAffine +
af::interpret), for the int8 GEMM parity tests on machines without
/root/reference. Run from the repo root: python tests/golden/make_int8_golden.py"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import oracle as O  # noqa: E402

cases = []
for (M, K, N, seed) in [(5, 40, 7, 1), (64, 160, 48, 2), (130, 96, 257, 3)]:
    rng = np.random.default_rng(seed)
    a = rng.integers(-128, 128, (M, K))
    b = rng.integers(-128, 128, (K, N))
    g = {"tensors": [{"id": "a", "shape": [M, K], "dtype": "i8"},
                     {"id": "b", "shape": [K, N], "dtype": "i8"},
                     {"id": "c", "shape": [M, N], "dtype": "i32"}],
         "ops": [{"op": "matmul", "inputs": ["a", "b"], "output": "c"}]}
    out = O.ref_run(json.dumps(g), {"a": a, "b": b}, "interpret")["%c"]
    cases.append({"name": f"i8_matmul_{M}x{K}x{N}", "graph": g, "a": a.tolist(), "b": b.tolist(),
                  "c": np.asarray(out, dtype=np.int64).tolist()})
# i8 NCHW conv graphs (the reference's conv2d lowering, i32 out)
conv_cases = []
for (B, C, H, W, OC, K, s, pad, seed) in [(1, 16, 5, 5, 8, 3, 1, "same", 4),
                                          (2, 64, 9, 8, 32, 3, 2, "valid", 5),
                                          (1, 32, 6, 6, 16, 1, 1, "valid", 6)]:
    rng = np.random.default_rng(seed)
    x = rng.integers(-128, 128, (B, C, H, W))
    w = rng.integers(-128, 128, (OC, C, K, K))
    OH = (H + s - 1) // s if pad == "same" else (H - K) // s + 1
    OW = (W + s - 1) // s if pad == "same" else (W - K) // s + 1
    g = {"tensors": [{"id": "x", "shape": [B, C, H, W], "dtype": "i8"},
                     {"id": "w", "shape": [OC, C, K, K], "dtype": "i8"},
                     {"id": "y", "shape": [B, OC, OH, OW], "dtype": "i32"}],
         "ops": [{"op": "conv2d", "inputs": ["x", "w"], "output": "y",
                  "attrs": {"stride": s, "padding": pad}}]}
    out = O.ref_run(json.dumps(g), {"x": x, "w": w}, "interpret")["%y"]
    conv_cases.append({"name": f"i8_conv_{B}x{C}x{H}x{W}_{OC}k{K}s{s}_{pad}", "graph": g,
                       "x": x.tolist(), "w": w.tolist(), "stride": s, "padding": pad,
                       "y": np.asarray(out, dtype=np.int64).tolist()})
json.dump({"generator": "tests/golden/make_int8_golden.py", "reference": "oracle/_ref af::interpret",
           "cases": cases, "conv_cases": conv_cases},
          open(os.path.join(os.path.dirname(__file__), "int8_matmul.json"), "w"))
print("wrote", len(cases), "cases")
