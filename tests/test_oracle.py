"""CPU tests: pin the oracle restatement (oracle/oracle.c) against the
reference's own known answers (tests/golden/kats.json, from test_interp.cpp)
and the reference's outputs on its own test graphs (tests/golden/
reference_graphs.json, generated from the compiled reference), and — where
the reference build oracle/_ref is present — against the live reference."""
import json
import math
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
KATS = json.load(open(os.path.join(GOLD, "kats.json")))
GRAPHS = json.load(open(os.path.join(GOLD, "reference_graphs.json")))["cases"]
CASES = {c["name"]: c for c in GRAPHS}


def dec(e):
    a = np.array([np.nan if v is None else v for v in e["data"]], dtype=np.float64)
    for i, s in e.get("nonfinite", {}).items():
        a[int(i)] = np.inf if s == "inf" else -np.inf
    return a.reshape(e["shape"])


needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


# ------------------------------------------------------------------ KATs ---

def test_f16_rne_kats():
    for x, want in KATS["f16_rne"]["cases"]:
        want = math.inf if want == "inf" else want
        assert O.round_f16(x) == want


def test_matmul_2x2_identity_kat():
    k = KATS["matmul_2x2_identity"]
    A = np.array(k["A"], float).reshape(2, 2)
    B = np.array(k["B"], float).reshape(2, 2)
    C = O.matmul(A, B, interp=True)
    assert C.ravel().tolist() == k["C"]


def test_mma_16x16x16_kat():
    # C = round_f32(sum_k f16(A) f16(B)) in double (test_interp.cpp:221-255)
    A = O.random_tensor((16, 16), "%A", 7)
    B = O.random_tensor((16, 16), "%B", 7)
    A16, B16 = O.round_to(A, O.F16), O.round_to(B, O.F16)
    want = np.zeros((16, 16))
    for i in range(16):
        for j in range(16):
            want[i, j] = O.round_to(np.array([sum(A16[i, k] * B16[k, j] for k in range(16))]),
                                    O.F32)[0]
    got = O.matmul(A16, B16)  # double accumulation, rounded f32 once
    assert np.array_equal(got, want)


def test_compare_profiles_kat():
    k = KATS["compare_profiles"]
    a, c = np.array(k["a"]), np.array(k["c"])
    ok, ma, mr, w = O.compare(a, a, k["F32"])
    assert ok and ma == 0.0
    ok, ma, mr, w = O.compare(a, c, k["F32"])
    assert not ok and w == k["worst_index"]
    assert not O.compare(a, c, k["Int"])[0]
    assert not O.compare(a, np.array([1.0, np.inf, 3.0]), 1.0)[0]  # non-finite fails


def test_conv_geometry_same_s2_even_has_zero_begin_pad():
    k = KATS["conv_same_s2_even_pad_begin_zero"]
    oh, ow, py, px = O.conv_geometry(k["inH"], k["inH"], k["k"], k["k"], (2, 2), (1, 1), True)
    assert oh == k["outH"] and py == k["padY"]


def test_gelu_tanh_closed_form_matches_reference_composite():
    c = CASES["mm_bias_gelu_32x24x16"]
    ins = {k: dec(v) for k, v in c["inputs"].items()}
    a, b, bias = (O.round_to(ins[n], O.F32) for n in ("a", "b", "bias"))
    y = O.matmul(a, b, bias, epi=O.EPI_GELU_TANH, interp=True)
    ref = dec(c["interpret"]["%y"])
    ok, ma, mr, _ = O.compare(y, ref, 1e-5)
    assert ok, (ma, mr)


# --------------------------------------------------- fixtures: restatement ---

def test_random_inputs_match_reference_generator():
    for c in GRAPHS:
        g = c["graph"]
        mine = O.random_graph_inputs(g, c["seed"], c["lo"], c["hi"])
        for tid, arr in mine.items():
            if tid in c.get("fixed", []):
                continue
            assert np.array_equal(arr, dec(c["inputs"][tid])), (c["name"], tid)


def test_matmul_interp_restatement_bit_exact():
    for name in ("matmul_4x4", "mm_bias_relu_48x40x24", "mm_bias_16x64x32"):
        c = CASES[name]
        ins = {k: O.round_to(dec(v), O.F32) for k, v in c["inputs"].items()}
        if name == "matmul_4x4":
            got = O.matmul(ins["a"], ins["b"], interp=True)
            want = dec(c["interpret"]["%c"])
        else:
            epi = O.EPI_RELU if "relu" in name else O.EPI_BIAS
            got = O.matmul(ins["a"], ins["b"], ins["bias"], epi=epi, interp=True)
            want = dec(c["interpret"]["%y" if "relu" in name else "%cb"])
        assert np.array_equal(got, want), name


def test_softmax_restatement():
    c = CASES["softmax_2x3"]
    x = O.round_to(dec(c["inputs"]["x"]), O.F32)
    got = O.round_to(O.softmax(x), O.F32)
    assert np.array_equal(got, dec(c["oracle"]["%y"]))
    assert O.compare(got, dec(c["interpret"]["%y"]), 1e-6)[0]


def test_conv_restatement_bit_exact_vs_convReference():
    for name in ("conv_direct", "conv_stride2", "conv_dil2", "conv_same", "conv_same_s2",
                 "conv_transposed_s2", "conv_transposed_same"):
        c = CASES[name]
        op = c["graph"]["ops"][0]
        at = op.get("attrs", {})
        s = at.get("stride", 1)
        d = at.get("dilation", 1)
        s, d = (s, s) if isinstance(s, int) else s, (d, d) if isinstance(d, int) else d
        x = O.round_to(dec(c["inputs"]["in"]), O.F32)
        w = O.round_to(dec(c["inputs"]["w"]), O.F32)
        tr = at.get("transposed", False)
        geo = O.conv_geometry(x.shape[2], x.shape[3], w.shape[2], w.shape[3], s, d,
                              at.get("padding") == "same", tr)
        y = O.conv_nchw(x, w, s, d, (geo[2], geo[3]), tr, (geo[0], geo[1]))
        assert np.array_equal(y, dec(c["oracle"]["%out"])), name
        assert O.compare(y, dec(c["interpret"]["%out"]), 1e-6)[0], name


def test_conv_nhwc_restatement_matches_reference_nhwc_graphs():
    for name, stride, pad in (("nhwc_conv3x3_same_relu", 1, 1),
                              ("nhwc_conv3x3_s2_prepadded_relu", 2, 0)):
        c = CASES[name]
        ins = {k: O.round_to(dec(v), O.F32) for k, v in c["inputs"].items()}
        w_ohwi = np.transpose(ins["w"], (0, 2, 3, 1))
        y = O.conv_nhwc(ins["x"], w_ohwi, ins["bias"], (stride, stride), (pad, pad),
                        epi=O.EPI_RELU)
        ok, ma, mr, _ = O.compare(y, dec(c["interpret"]["%y"]), 1e-6)
        assert ok, (name, ma, mr)


def test_batch_matmul_restatement():
    c = CASES["batch_matmul"]
    got = O.batch_matmul(O.round_to(dec(c["inputs"]["x"]), O.F32),
                         O.round_to(dec(c["inputs"]["y"]), O.F32))
    assert np.array_equal(got, dec(c["oracle"]["%z"]))


def test_attention_restatement_vs_reference_graphs():
    for name, causal in (("attention_1x2x8x4", False), ("attn_f16_1x2x16x8", False),
                         ("attn_f16_causal_1x2x16x8", True)):
        c = CASES[name]
        t = O.F16 if "f16" in name else O.F32
        q, k, v = (O.round_to(dec(c["inputs"][n]), t) for n in ("q", "k", "v"))
        bias = O.round_to(dec(c["inputs"]["bias"]), O.F32) if "bias" in c["inputs"] else None
        o = O.attention(q, k, v, bias=bias, causal=causal)
        ok, ma, mr, _ = O.compare(o, dec(c["interpret"]["%out"]), 1e-6)
        assert ok, (name, ma, mr)


def test_layernorm_restatement_properties():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((5, 64))
    r = rng.standard_normal((5, 64))
    y, s = O.layernorm(x, r, np.ones(64), np.zeros(64), 1e-12)
    assert np.allclose(s, x + r)
    assert np.allclose(y.mean(-1), 0, atol=1e-12)
    assert np.allclose(y.var(-1), 1, atol=1e-9)


# -------------------------------------------------- live reference (_ref) ---

@needs_ref
def test_live_reference_hash_rounding_compare():
    L = O.ref_lib()
    for s in ("%a", "%bias", "%some_long_buffer_name_17", ""):
        assert O.std_hash(s) == L.afref_std_hash(s.encode())
    xs = np.random.default_rng(1).standard_normal(2000) * 1e3
    xs = np.concatenate([xs, [65504.0, 65520.0, 1e-8, -6e-5, 2.0**-24, 3 * 2.0**-26]])
    for t in (O.F32, O.F16, O.I8, O.I32):
        mine = O.round_to(xs, t)
        theirs = np.array([L.afref_round_to_type(float(v), t) for v in xs])
        assert np.array_equal(mine, theirs), t
    a = xs[:100]
    b = a * (1 + 1e-7)
    assert O.compare(a, b, 1e-6)[:3] == O.ref_compare(a, b, "F32")[:3]


@needs_ref
def test_live_reference_reproduces_committed_fixtures():
    for c in GRAPHS[:6]:
        ins = {k: dec(v) for k, v in c["inputs"].items()}
        out = O.ref_run(json.dumps(c["graph"]), ins, "interpret")
        for k, v in c["interpret"].items():
            assert np.array_equal(out[k], dec(v)), (c["name"], k)


# ------------------------------------------------------------- int8 path ---

I8 = json.load(open(os.path.join(GOLD, "int8_matmul.json")))["cases"]


def test_quantize_kat():
    # test_interp.cpp:286-307: quant scale 0.5 -> {1, -2, 127, -1}
    assert O.quantize([0.74, -0.76, 100.0, -0.25], 0.5).tolist() == [1, -2, 127, -1]


def test_int8_matmul_restatement_vs_reference_fixtures():
    for c in I8:
        a, b = np.array(c["a"]), np.array(c["b"])
        got = O.matmul_i8(a, b.T)
        assert np.array_equal(got, np.array(c["c"])), c["name"]


def test_int8_requant_rounding_half_away():
    acc_a = np.array([[1, 1, 1]])
    b = np.array([[1, 0, 0], [1, 1, 1], [-1, -1, -1]])  # acc = 1, 3, -3
    got = O.matmul_i8(acc_a, b, mode=1, scale=0.5)  # 0.5 -> 1, 1.5 -> 2, -1.5 -> -2
    assert got.tolist() == [[1, 2, -2]]
    assert O.matmul_i8(np.full((1, 64), 127), np.full((1, 64), 127), mode=1, scale=1.0).tolist() == [[127]]


@needs_ref
def test_int8_matmul_restatement_vs_live_reference():
    rng = np.random.default_rng(7)
    M, K, N = 9, 72, 11
    a, b = rng.integers(-128, 128, (M, K)), rng.integers(-128, 128, (K, N))
    g = {"tensors": [{"id": "a", "shape": [M, K], "dtype": "i8"},
                     {"id": "b", "shape": [K, N], "dtype": "i8"},
                     {"id": "c", "shape": [M, N], "dtype": "i32"}],
         "ops": [{"op": "matmul", "inputs": ["a", "b"], "output": "c"}]}
    out = O.ref_run(json.dumps(g), {"a": a, "b": b}, "interpret")["%c"]
    assert np.array_equal(O.matmul_i8(a, b.T), out)


def _pad_of(c, K):
    return (K // 2, K // 2) if c["padding"] == "same" else (0, 0)


def test_int8_conv_restatement_vs_reference_fixtures():
    for c in json.load(open(os.path.join(GOLD, "int8_matmul.json")))["conv_cases"]:
        x = np.transpose(np.array(c["x"]), (0, 2, 3, 1))
        w = np.transpose(np.array(c["w"]), (0, 2, 3, 1))
        K = w.shape[1]
        y = np.array(c["y"])
        got = O.conv_i8(x, w, stride=(c["stride"],) * 2, pad=_pad_of(c, K),
                        out_hw=(y.shape[2], y.shape[3]))
        assert np.array_equal(np.transpose(got, (0, 3, 1, 2)), y), c["name"]
