"""Graph builders in the reference's unchanged graph-JSON API
(frontend.cpp:57-113) for the BASELINE patterns. Test /
bench infrastructure (used by tests/golden/make_golden.py and bench.py's
reference arm)."""
import math

import numpy as np

from . import conv_geometry


def T(id_, shape, dtype=None):
    d = {"id": id_, "shape": list(shape)}
    if dtype:
        d["dtype"] = dtype
    return d


def conv_graph(attrs, in_shape, w_shape, out_shape):
    return {"tensors": [T("in", in_shape), T("w", w_shape), T("out", out_shape)],
            "ops": [{"op": "conv2d", "inputs": ["in", "w"], "output": "out", "attrs": attrs}]}


def matmul_epi_graph(M, N, K, act):
    """matmul -> broadcast_in_dim(bias) -> add -> act, SURVEY.md App. B."""
    tensors = [T("a", [M, K]), T("b", [K, N]), T("bias", [N]), T("c", [M, N]), T("bb", [M, N]),
               T("cb", [M, N])]
    ops = [{"op": "matmul", "inputs": ["a", "b"], "output": "c"},
           {"op": "broadcast_in_dim", "inputs": ["bias"], "output": "bb", "attrs": {"dims": [1]}},
           {"op": "add", "inputs": ["c", "bb"], "output": "cb"}]
    fixed = {}
    if act == "relu":
        tensors += [T("z", [M, N]), T("y", [M, N])]
        ops += [{"op": "max", "inputs": ["cb", "z"], "output": "y"}]
        fixed["z"] = np.zeros((M, N))
    elif act == "gelu":
        # tanh-GELU composite: x * sigmoid(2u), sigmoid via softmax([2u, 0])[0]
        x = "cb"
        tensors += [T("c1", [M, N]), T("c2", [M, N]), T("mask", [M, N, 2]), T("x2", [M, N]),
                    T("x3", [M, N]), T("t", [M, N]), T("s", [M, N]), T("u2", [M, N]),
                    T("bu", [M, N, 2]), T("m", [M, N, 2]), T("sm", [M, N, 2]),
                    T("sel", [M, N, 2]), T("sg", [M, N]), T("y", [M, N])]
        ops += [{"op": "mul", "inputs": [x, x], "output": "x2"},
                {"op": "mul", "inputs": ["x2", x], "output": "x3"},
                {"op": "mul", "inputs": ["x3", "c1"], "output": "t"},
                {"op": "add", "inputs": [x, "t"], "output": "s"},
                {"op": "mul", "inputs": ["s", "c2"], "output": "u2"},
                {"op": "broadcast_in_dim", "inputs": ["u2"], "output": "bu",
                 "attrs": {"dims": [0, 1]}},
                {"op": "mul", "inputs": ["bu", "mask"], "output": "m"},
                {"op": "softmax", "inputs": ["m"], "output": "sm", "attrs": {"axis": -1}},
                {"op": "mul", "inputs": ["sm", "mask"], "output": "sel"},
                {"op": "reduce", "inputs": ["sel"], "output": "sg",
                 "attrs": {"op": "sum", "axis": 2}},
                {"op": "mul", "inputs": [x, "sg"], "output": "y"}]
        fixed["c1"] = np.full((M, N), 0.044715)
        fixed["c2"] = np.full((M, N), 2.0 * math.sqrt(2.0 / math.pi))
        mask = np.zeros((M, N, 2))
        mask[..., 0] = 1.0
        fixed["mask"] = mask
    return {"tensors": tensors, "ops": ops}, fixed


def attention_graph(B, H, N, D, causal, dtype="f16"):
    g = {"tensors": [T("q", [B, H, N, D], dtype), T("k", [B, H, N, D], dtype),
                     T("kt", [B, H, D, N], dtype), T("v", [B, H, N, D], dtype),
                     T("qk", [B, H, N, N]), T("soft", [B, H, N, N]), T("out", [B, H, N, D])],
         "ops": [{"op": "transpose", "inputs": ["k"], "output": "kt",
                  "attrs": {"perm": [0, 1, 3, 2]}},
                 {"op": "batch_matmul", "inputs": ["q", "kt"], "output": "qk"}]}
    fixed = {}
    src = "qk"
    if causal:
        g["tensors"] += [T("mask", [B, H, N, N]), T("qkb", [B, H, N, N])]
        g["ops"].append({"op": "add", "inputs": ["qk", "mask"], "output": "qkb"})
        m = np.zeros((B, H, N, N))
        m[..., np.triu_indices(N, 1)[0], np.triu_indices(N, 1)[1]] = -np.inf
        fixed["mask"] = m
        src = "qkb"
    g["ops"] += [{"op": "softmax", "inputs": [src], "output": "soft", "attrs": {"axis": -1}},
                 {"op": "batch_matmul", "inputs": ["soft", "v"], "output": "out"}]
    return g, fixed


def nhwc_conv_graph(B, H, W, C, OC, k, stride, padding):
    """transpose(NHWC->NCHW) -> conv2d -> bias -> max(zeros) -> transpose back."""
    geo = conv_geometry(H, W, k, k, (stride, stride), (1, 1), padding == "same")
    OH, OW = geo[0], geo[1]
    g = {"tensors": [T("x", [B, H, W, C]), T("xt", [B, C, H, W]), T("w", [OC, C, k, k]),
                     T("bias", [OC]), T("c", [B, OC, OH, OW]), T("bb", [B, OC, OH, OW]),
                     T("cb", [B, OC, OH, OW]), T("z", [B, OC, OH, OW]), T("r", [B, OC, OH, OW]),
                     T("y", [B, OH, OW, OC])],
         "ops": [{"op": "transpose", "inputs": ["x"], "output": "xt",
                  "attrs": {"perm": [0, 3, 1, 2]}},
                 {"op": "conv2d", "inputs": ["xt", "w"], "output": "c",
                  "attrs": {"padding": padding, "stride": stride}},
                 {"op": "broadcast_in_dim", "inputs": ["bias"], "output": "bb",
                  "attrs": {"dims": [1]}},
                 {"op": "add", "inputs": ["c", "bb"], "output": "cb"},
                 {"op": "max", "inputs": ["cb", "z"], "output": "r"},
                 {"op": "transpose", "inputs": ["r"], "output": "y",
                  "attrs": {"perm": [0, 2, 3, 1]}}]}
    return g, {"z": np.zeros((B, OC, OH, OW))}


