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
json.dump({"generator": "tests/golden/make_int8_golden.py", "reference": "oracle/_ref af::interpret",
           "cases": cases}, open(os.path.join(os.path.dirname(__file__), "int8_matmul.json"), "w"))
print("wrote", len(cases), "cases")
