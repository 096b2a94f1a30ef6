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




def bert_layer_graph(S, hidden, heads, ffn):
    """A BERT-base-style encoder layer (one sequence) in the unchanged graph
    API, as SURVEY.md App. B writes it: Q/K/V projections as three matmuls +
    bias, heads via reshape + transpose, scaled attention (constant-tensor
    mul), output projection + bias + residual, GELU FFN (the 14-nest
    composite) + residual. Layernorm has no expression in the reference API
    (frontend.cpp:153-157) and is omitted. Returns (graph, fixed constants)."""
    dh = hidden // heads
    t, ops, fixed = [], [], {}

    def ten(i, s):
        t.append(T(i, s))

    def op(o, ins, out, **attrs):
        d = {"op": o, "inputs": ins, "output": out}
        if attrs:
            d["attrs"] = attrs
        ops.append(d)

    def linear(x, w, b, out, k, n):
        ten(w, [k, n]), ten(b, [n]), ten(out + "_mm", [S, n]), ten(out + "_bb", [S, n]), ten(out, [S, n])
        op("matmul", [x, w], out + "_mm")
        op("broadcast_in_dim", [b], out + "_bb", dims=[1])
        op("add", [out + "_mm", out + "_bb"], out)

    ten("x", [S, hidden])
    for p in ("q", "k", "v"):
        linear("x", "w" + p, "b" + p, p, hidden, hidden)
        ten(p + "4", [1, S, heads, dh]), ten(p + "h", [1, heads, S, dh])
        op("reshape", [p], p + "4")
        op("transpose", [p + "4"], p + "h", perm=[0, 2, 1, 3])
    ten("kt", [1, heads, dh, S]), ten("qk", [1, heads, S, S]), ten("sc", [1, heads, S, S])
    ten("qs", [1, heads, S, S]), ten("soft", [1, heads, S, S]), ten("ctx", [1, heads, S, dh])
    op("transpose", ["kh"], "kt", perm=[0, 1, 3, 2])
    op("batch_matmul", ["qh", "kt"], "qk")
    op("mul", ["qk", "sc"], "qs")
    op("softmax", ["qs"], "soft", axis=-1)
    op("batch_matmul", ["soft", "vh"], "ctx")
    fixed["sc"] = np.full((1, heads, S, S), 1.0 / math.sqrt(dh))
    ten("ctx_t", [1, S, heads, dh]), ten("ctx2", [S, hidden])
    op("transpose", ["ctx"], "ctx_t", perm=[0, 2, 1, 3])
    op("reshape", ["ctx_t"], "ctx2")
    linear("ctx2", "wo", "bo", "attn", hidden, hidden)
    ten("res1", [S, hidden])
    op("add", ["x", "attn"], "res1")
    linear("res1", "w1", "b1", "h", hidden, ffn)
    # tanh-GELU composite on h
    for i, s in [("c1", [S, ffn]), ("c2", [S, ffn]), ("mask", [S, ffn, 2]), ("x2", [S, ffn]),
                 ("x3", [S, ffn]), ("tt", [S, ffn]), ("ss", [S, ffn]), ("u2", [S, ffn]),
                 ("bu", [S, ffn, 2]), ("mm", [S, ffn, 2]), ("sm", [S, ffn, 2]),
                 ("sel", [S, ffn, 2]), ("sg", [S, ffn]), ("g", [S, ffn])]:
        ten(i, s)
    op("mul", ["h", "h"], "x2")
    op("mul", ["x2", "h"], "x3")
    op("mul", ["x3", "c1"], "tt")
    op("add", ["h", "tt"], "ss")
    op("mul", ["ss", "c2"], "u2")
    op("broadcast_in_dim", ["u2"], "bu", dims=[0, 1])
    op("mul", ["bu", "mask"], "mm")
    op("softmax", ["mm"], "sm", axis=-1)
    op("mul", ["sm", "mask"], "sel")
    op("reduce", ["sel"], "sg", op="sum", axis=2)
    op("mul", ["h", "sg"], "g")
    fixed["c1"] = np.full((S, ffn), 0.044715)
    fixed["c2"] = np.full((S, ffn), 2.0 * math.sqrt(2.0 / math.pi))
    m = np.zeros((S, ffn, 2))
    m[..., 0] = 1.0
    fixed["mask"] = m
    linear("g", "w2", "b2", "o2", ffn, hidden)
    ten("y", [S, hidden])
    op("add", ["res1", "o2"], "y")
    flops = 2.0 * S * hidden * (4 * hidden + 2 * ffn) + 4.0 * heads * S * S * dh
    return {"tensors": t, "ops": ops, "outputs": ["y"]}, fixed, flops
