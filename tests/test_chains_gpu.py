"""GPU parity of the memory-bound chains (K4 softmax, K5 residual+layernorm,
elementwise / reduce / transpose / convert) and of the device-side input
generator against the reference's makeRandomTensor.

Tolerances: fp32 chains 1e-5; fp16 output one fp16 ulp (2^-10); bf16 output
one bf16 ulp (2^-7), in the reference's max(|a|,|b|,1) rule."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2603_06731_b200 import BinOp, ReduceKind, ops
from tests.gpu_util import check, seeded, to_host

pytestmark = pytest.mark.gpu


def test_fill_uniform_bit_exact_vs_reference_generator(cuda):
    for dt, code in ((torch.float32, O.F32), (torch.float16, O.F16), (torch.bfloat16, O.BF16)):
        s0 = O.stream_seed("%a", 11)
        x = ops.fill_uniform((1000, 3), s0, -1.0, 1.0, dtype=dt)
        want = O.round_to(O.random_tensor((1000, 3), "%a", 11, -1.0, 1.0), code)
        assert np.array_equal(to_host(x), want), dt


@pytest.mark.parametrize("rows,cols,dt,od,tol", [
    (1000, 2048, torch.float16, torch.float16, 2.0**-10),
    (5003, 2048, torch.float16, torch.float16, 2.0**-10),  # TMA-streamed kernel
    (6000, 512, torch.bfloat16, torch.bfloat16, 2.0**-7),  # TMA-streamed, short rows
    (257, 512, torch.float32, torch.float32, 1e-5),
    (64, 8192, torch.float16, torch.float32, 1e-5),  # > 4096 cols: block kernel
    (5, 100, torch.bfloat16, torch.bfloat16, 2.0**-7),
    (3, 7, torch.float32, torch.float32, 1e-5),  # ragged: non-vector path
])
def test_softmax(cuda, rows, cols, dt, od, tol):
    x, xh = seeded((rows, cols), "x", 12, -4.0, 4.0, dtype=dt)
    y = ops.softmax(x, out_dtype=od)
    want = O.round_to(O.softmax(xh), {torch.float32: O.F32, torch.float16: O.F16,
                                      torch.bfloat16: O.BF16}[od])
    check(to_host(y), want, tol, "softmax")


def test_softmax_full_size_streamed_repeat(cuda):
    # BASELINE's softmax workload at full size ([8*16*2048, 2048] fp16, 1772 rows
    # per SM through the TMA ring), launched repeatedly: an early pass of a
    # ring-slot wait shows up as corrupted rows or a hang. Checked against the
    # oracle's softmaxReference restatement on sampled rows of the same fp16
    # values (1 fp16 ulp).
    g = torch.Generator(device="cuda").manual_seed(5)
    x = (torch.rand((262144, 2048), generator=g, device="cuda") * 8 - 4).half()
    rows = torch.arange(0, 262144, 4099, device="cuda")
    want = O.round_to(O.softmax(to_host(x[rows])), O.F16)
    for _ in range(4):
        y = ops.softmax(x)
        check(to_host(y[rows]), want, 2.0**-10, "softmax full size")


def test_layernorm_full_size_streamed_repeat(cuda):
    # BERT's residual + layernorm at full size ([64*512, 768] bf16) repeatedly,
    # against the oracle's layernorm restatement on sampled rows (1 bf16 ulp).
    g = torch.Generator(device="cuda").manual_seed(6)
    x = (torch.rand((32768, 768), generator=g, device="cuda") * 2 - 1).bfloat16()
    r = (torch.rand((32768, 768), generator=g, device="cuda") * 2 - 1).bfloat16()
    gam = torch.rand(768, generator=g, device="cuda") * 0.2 + 0.9
    bet = torch.rand(768, generator=g, device="cuda") * 0.2 - 0.1
    rows = torch.arange(0, 32768, 331, device="cuda")
    want = O.round_to(O.layernorm(to_host(x[rows]), to_host(r[rows]), to_host(gam), to_host(bet),
                                  1e-12)[0], O.BF16)
    for _ in range(4):
        y = ops.layernorm_residual(x, r, gam, bet, eps=1e-12)
        check(to_host(y[rows]), want, 2.0**-7, "layernorm full size")


def test_softmax_large_magnitudes_finite(cuda):
    # rows with entries up to 80 in magnitude stay finite
    x = torch.linspace(-80, 80, 4096, device="cuda").reshape(4, 1024)
    y = ops.softmax(x)
    assert torch.isfinite(y).all()
    check(to_host(y), O.softmax(to_host(x)), 1e-5, "softmax |x|<=80")


@pytest.mark.parametrize("rows,cols,dt,tol", [
    (1024, 768, torch.bfloat16, 2.0**-7),
    (9001, 768, torch.bfloat16, 2.0**-7),  # TMA-streamed kernel (rows >= 8 per SM)
    (5000, 1024, torch.float16, 2.0**-10),
    (100, 768, torch.float32, 1e-5),
    (33, 1024, torch.float16, 2.0**-10),
    (7, 5000, torch.float32, 1e-5),  # block kernel
])
def test_layernorm_residual(cuda, rows, cols, dt, tol):
    x, xh = seeded((rows, cols), "x", 13, dtype=dt)
    r, rh = seeded((rows, cols), "r", 13, dtype=dt)
    g, gh = seeded((cols,), "g", 13, 0.9, 1.1, dtype=torch.float32)
    b, bh = seeded((cols,), "be", 13, -0.1, 0.1, dtype=torch.float32)
    s = torch.empty_like(x)
    y = ops.layernorm_residual(x, r, g, b, eps=1e-12, sum_out=s)
    code = {torch.float32: O.F32, torch.float16: O.F16, torch.bfloat16: O.BF16}[dt]
    want_y, want_s = O.layernorm(xh, rh, gh, bh, 1e-12)
    check(to_host(y), O.round_to(want_y, code), tol, "layernorm y")
    check(to_host(s), O.round_to(want_s, code), tol, "layernorm sum")


def test_elementwise_reduce_transpose(cuda):
    a, ah = seeded((3, 5), "a", 31, dtype=torch.float32)
    b, bh = seeded((3, 5), "b", 31, dtype=torch.float32)
    for op, fn in ((BinOp.ADD, np.add), (BinOp.SUB, np.subtract), (BinOp.MUL, np.multiply),
                   (BinOp.MAX, np.maximum)):
        got = to_host(ops.elementwise(a, b, op))
        assert np.array_equal(got, O.round_to(fn(ah, bh), O.F32)), op
    e = to_host(ops.elementwise(a, None, BinOp.EXP))
    check(e, O.round_to(np.exp(ah), O.F32), 1e-6, "exp")
    bias, biash = seeded((5,), "bias", 31, dtype=torch.float32)
    got = to_host(ops.elementwise(a, bias, BinOp.ADD, b_period=5))
    assert np.array_equal(got, O.round_to(ah + biash[None, :], O.F32))
    assert np.array_equal(to_host(ops.reduce_lastdim(a, ReduceKind.MAX)), ah.max(-1))
    check(to_host(ops.reduce_lastdim(a, ReduceKind.SUM)), ah.sum(-1), 1e-6, "reduce sum")
    x, xh = seeded((2, 3, 4, 5), "x", 33, dtype=torch.float32)
    assert np.array_equal(to_host(ops.transpose(x, (0, 3, 1, 2))), xh.transpose(0, 3, 1, 2))
    h = ops.convert(x, torch.float16)
    assert np.array_equal(to_host(h), O.round_to(xh, O.F16))


@pytest.mark.parametrize("pool", ["0", "3", "16"])
def test_stream_row_pool(cuda, pool):
    # the streamed kernels with 1/3 or 1/16 of the rows claimed dynamically
    # (and fully static): skip / end markers, claims, no residual, repeated
    # launches on one stream (the pool counter resets per launch)
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, AFG_STREAM_POOL=pool)
    out = subprocess.run([sys.executable, os.path.join(here, "stream_pool_check.py")], env=env,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]


def test_concurrent_streams_row_pool(cuda):
    # the softmax tail pool keeps one counter pair per stream: concurrent
    # launches on two streams each match their single-stream result exactly
    g = torch.Generator(device="cuda").manual_seed(17)
    xs = [(torch.rand((40000, 2048), generator=g, device="cuda") * 8 - 4).half() for _ in range(2)]
    want = [ops.softmax(x) for x in xs]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for _ in range(5):
        got = []
        for s, x in zip(streams, xs):
            with torch.cuda.stream(s):
                got.append(ops.softmax(x))
        torch.cuda.synchronize()
        for a, b in zip(got, want):
            assert torch.equal(a, b)
