"""GPU parity of K1 (tcgen05 bf16/fp16 GEMM + fused epilogue) and K1b (fp32
SIMT GEMM) against the oracle restatement of the reference path.

Tolerances (the reference's rule |a-b| <= tol * max(|a|,|b|,1),
interp.cpp:698-730):
  * fp32 GEMM vs the interpreter restatement (sequential f32-rounded FMA,
    interp.cpp:335-347): bit-exact (tol 0); vs the double oracle
    (matmulReference, oracles.cpp:122-134): 1e-4 (BASELINE north star).
  * bf16/fp16 inputs, fp32 output, vs the double oracle on the same rounded
    inputs: 1e-5 for K <= 1024; for longer K the forward-error bound of fp32
    (tensor-core) accumulation, |C - C_exact| <= 2^-19 * sum_k |a_ik b_kj|
    (measured 7e-7 of sum|ab| at K = 8192).
  * bf16/fp16 output: one output ulp, 2^-7 (bf16) / 2^-10 (fp16), against the
    oracle result rounded to the output type.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2603_06731_b200 import Epilogue, Layout, ops
from tests.gpu_util import check, seeded, to_host

pytestmark = pytest.mark.gpu

EPI = {Epilogue.NONE: O.EPI_NONE, Epilogue.BIAS: O.EPI_BIAS, Epilogue.BIAS_RELU: O.EPI_RELU,
       Epilogue.BIAS_GELU_TANH: O.EPI_GELU_TANH, Epilogue.BIAS_GELU_ERF: O.EPI_GELU_ERF}
ULP = {torch.bfloat16: 2.0**-7, torch.float16: 2.0**-10}


def run_case(cuda, M, N, K, dt=torch.bfloat16, out=None, epi=Epilogue.BIAS_GELU_TANH,
             layout=Layout.B_KN, residual=False, seed=5, rows=None):
    out = out or dt
    a, ah = seeded((M, K), "a", seed, dtype=dt)
    bshape = (K, N) if layout == Layout.B_KN else (N, K)
    b, bh = seeded(bshape, "b", seed, dtype=dt)
    bias, biash = seeded((N,), "bias", seed, dtype=torch.float32)
    res = resh = None
    if residual:
        res, resh = seeded((M, N), "res", seed, dtype=out)
    c = ops.gemm(a, b, bias=bias if epi != Epilogue.NONE else None, epilogue=epi,
                 out_dtype=out, b_layout=layout, residual=res)
    torch.cuda.synchronize()
    got = to_host(c)
    if rows is not None:
        got = got[rows]
    out_code = O.F32 if out == torch.float32 else (O.BF16 if out == torch.bfloat16 else O.F16)
    # fp32 accumulation then the epilogue in double, rounded to the output type
    acc = O.matmul(ah, bh, biash, epi=EPI[epi], out_t=O.F64, b_nk=layout == Layout.B_NK,
                   rows=rows)
    if residual:
        acc = acc + (resh if rows is None else resh[rows])
    want = O.round_to(acc, out_code)
    what = f"gemm {M}x{N}x{K} {dt}->{out} epi={int(epi)}"
    if out in ULP:
        return check(got, want, ULP[out], what)
    if K <= 1024:
        return check(got, want, 1e-5, what)
    absab = O.matmul(np.abs(ah), np.abs(bh), b_nk=layout == Layout.B_NK, rows=rows)
    err = np.abs(got - want)
    bound = 2.0**-19 * absab + 1e-6
    assert (err <= bound).all(), f"{what}: max err/sum|ab| = {(err / absab).max():.3e}"
    return float((err / absab).max())


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 256), (100, 200, 72),
                                   (333, 130, 200), (1024, 1024, 1024), (257, 768, 768),
                                   (64, 64, 64), (2048, 2048, 512)])
def test_bf16_gelu_shapes(cuda, M, N, K):
    run_case(cuda, M, N, K)


@pytest.mark.parametrize("epi", list(Epilogue))
def test_bf16_epilogues_fp32_out(cuda, epi):
    run_case(cuda, 384, 320, 256, out=torch.float32, epi=epi)


def test_fp16_relu_fp16_out(cuda):
    run_case(cuda, 512, 512, 384, dt=torch.float16, epi=Epilogue.BIAS_RELU)


def test_b_nk_layout(cuda):
    run_case(cuda, 512, 384, 256, layout=Layout.B_NK)
    run_case(cuda, 300, 64, 128, layout=Layout.B_NK, epi=Epilogue.BIAS)


def test_residual_epilogue(cuda):
    run_case(cuda, 512, 768, 768, epi=Epilogue.BIAS, residual=True)


def test_large_k_fp32_out(cuda):
    run_case(cuda, 256, 256, 8192, out=torch.float32, epi=Epilogue.BIAS)


def test_benchmarked_16384_sampled_block(cuda):
    """The exact bench workload (BASELINE configs[1] at 16384^3, bf16 + bias +
    tanh-GELU, bf16 out, inputs from the device generator = the reference's
    makeRandomTensor stream) checked on a sampled block of rows x columns
    against the oracle on the same bf16 values (1 bf16 ulp)."""
    import oracle as Orc
    n = 16384
    A = ops.fill_uniform((n, n), Orc.stream_seed("%a", 1), -1, 1, torch.bfloat16)
    B = ops.fill_uniform((n, n), Orc.stream_seed("%b", 1), -1, 1, torch.bfloat16)
    bias = ops.fill_uniform((n,), Orc.stream_seed("%bias", 1), -1, 1, torch.float32)
    C = ops.gemm(A, B, bias=bias, epilogue=Epilogue.BIAS_GELU_TANH)
    torch.cuda.synchronize()
    rows = torch.tensor([0, 1, 255, 256, 8191, 12345, 16383])
    cols = torch.tensor(list(range(0, 64)) + [4095, 4096, 9999, 16383])
    a = to_host(A[rows.cuda()])
    b = to_host(B[:, cols.cuda()])
    want = Orc.round_to(Orc.matmul(a, b, to_host(bias[cols.cuda()]), epi=Orc.EPI_GELU_TANH,
                                   out_t=Orc.F64), Orc.BF16)
    got = to_host(C[rows.cuda()][:, cols.cuda()])
    check(got, want, 2.0**-7, "bench gemm 16384^3 sampled block")
    del A, B, C
    torch.cuda.empty_cache()


def test_full_size_sampled_rows_4096(cuda):
    # BASELINE configs[1] shape class at full size, parity on sampled rows
    rows = np.array([0, 1, 127, 128, 2047, 2048, 4000, 4095])
    run_case(cuda, 4096, 4096, 4096, rows=rows)


# ------------------------------------------------------------------- fp32 ---

def test_fp32_config1_bit_exact_vs_interpreter(cuda):
    """BASELINE configs[0]: fp32 1024^3 + bias + ReLU, the reference's own
    matmul->broadcast_in_dim->add->max graph. Sequential fp32 FMA == the
    interpreter's double FMA rounded to f32 at every store."""
    n = 1024
    a, ah = seeded((n, n), "a", 1, dtype=torch.float32)
    b, bh = seeded((n, n), "b", 2, dtype=torch.float32)
    bias, biash = seeded((n,), "bias", 3, dtype=torch.float32)
    c = ops.gemm(a, b, bias=bias, epilogue=Epilogue.BIAS_RELU)
    got = to_host(c)
    want_interp = O.matmul(ah, bh, biash, epi=O.EPI_RELU, interp=True)
    ok, ma, mr, w = O.compare(got, want_interp, 0.0)
    assert ok, f"not bit-exact vs interpreter: max_abs {ma} at {w}"
    want_ref = O.matmul(ah, bh, biash, epi=O.EPI_RELU, interp=False)
    check(got, want_ref, 1e-4, "fp32 vs double oracle")


def test_fp32_ragged(cuda):
    a, ah = seeded((37, 53), "a", 9, dtype=torch.float32)
    b, bh = seeded((53, 29), "b", 9, dtype=torch.float32)
    c = ops.gemm(a, b)
    assert np.array_equal(to_host(c), O.matmul(ah, bh, interp=True))


def test_batched_matmul(cuda):
    a, ah = seeded((2, 2, 3, 4), "x", 32, dtype=torch.float32)
    b, bh = seeded((2, 2, 4, 5), "y", 32, dtype=torch.float32)
    c = ops.gemm_batched(a, b)
    check(to_host(c), O.batch_matmul(ah, bh), 1e-6, "batch_matmul")


def test_unaligned_bf16_runs_simt_path(cuda):
    # K = 20 -> row pitch 40 B, not TMA-addressable: SIMT kernel, same contract
    run_case(cuda, 33, 40, 20, out=torch.float32, epi=Epilogue.BIAS_RELU)


def test_splitk_partials_and_epilogue_apply(cuda):
    """The split-K / TP path on one GPU: two K-slice fp32 partials (strided A
    views, lda = K) summed, then the standalone epilogue kernel."""
    from paper_2603_06731_b200 import lib
    from paper_2603_06731_b200.ops import _ptr, _stream
    M, N, K = 512, 384, 1024
    a, ah = seeded((M, K), "a", 11, dtype=torch.bfloat16)
    b, bh = seeded((K, N), "b", 11, dtype=torch.bfloat16)
    bias, biash = seeded((N,), "bias", 11, dtype=torch.float32)
    p0 = ops.gemm(a[:, : K // 2], b[: K // 2], out_dtype=torch.float32)
    p1 = ops.gemm(a[:, K // 2:], b[K // 2:], out_dtype=torch.float32)
    acc = p0 + p1
    c = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    assert lib().afg_epilogue_apply(_ptr(acc), _ptr(bias), None, _ptr(c), M, N, N,
                                    int(Epilogue.BIAS_GELU_TANH), 0, 2, _stream()) == 0
    want = O.round_to(O.matmul(ah, bh, biash, epi=O.EPI_GELU_TANH, out_t=O.F64), O.BF16)
    check(to_host(c), want, 2.0**-7, "split-K + epilogue")


@pytest.mark.parametrize("N,out", [(64, torch.bfloat16), (64, torch.float32), (128, torch.bfloat16),
                                   (256, torch.bfloat16)])
def test_many_tiles_per_cta(cuda, N, out):
    """>= 3 tiles per persistent CTA exercises the accumulator double-buffer
    hand-off (tmem full/empty phases) for every BLOCK_N / staging variant."""
    M = 148 * 128 * 3 + 77
    run_case(cuda, M, N, 128, out=out, epi=Epilogue.BIAS_RELU, rows=np.arange(0, M, 997))


# 256 x 256 tiles on a CTA pair (cta_group::2): BLOCK_N = 256 problems with
# K >= 768 and at least a wave of pair tiles. Ragged M / N / K, both B layouts,
# every output type, residual, >= 3 pair tiles per cluster (accumulator hand-off
# across both CTAs' epilogues), the 5-stage (K < 2048) and 6-stage variants,
# and both epilogue widths (GELU: four warp groups; bias / ReLU: two).
PAIR_ROWS = np.array([0, 127, 128, 255, 256, 2047, 3999])


@pytest.mark.parametrize("layout", [Layout.B_KN, Layout.B_NK])
@pytest.mark.parametrize("out", [torch.bfloat16, torch.float32])
def test_pair_tiles_ragged(cuda, layout, out):
    run_case(cuda, 4000, 2300, 800, out=out, layout=layout, rows=PAIR_ROWS)


def test_pair_tiles_fp16_residual(cuda):
    run_case(cuda, 4000, 4352, 1024, dt=torch.float16, epi=Epilogue.BIAS, residual=True,
             rows=PAIR_ROWS)


@pytest.mark.parametrize("epi", [Epilogue.BIAS_RELU, Epilogue.BIAS_GELU_ERF])
def test_pair_tiles_many_per_cluster(cuda, epi):
    M = 256 * 74 * 3 + 77
    run_case(cuda, M, 512, 768, epi=epi, layout=Layout.B_NK, rows=np.arange(0, M, 1013))


@pytest.mark.parametrize("epi", [Epilogue.BIAS, Epilogue.BIAS_GELU_TANH])
def test_pair_tiles_long_k(cuda, epi):
    run_case(cuda, 4000, 2300, 2112, epi=epi, rows=PAIR_ROWS)


def test_pair_tiles_bert_ffn1_sampled(cuda):
    """BERT FFN1 at full size (B64 x S512 tokens, 768 -> 3072, erf GELU)."""
    rows = np.array([0, 1, 255, 256, 16383, 32767])
    run_case(cuda, 32768, 3072, 768, epi=Epilogue.BIAS_GELU_ERF, layout=Layout.B_NK, rows=rows)


def test_round_sync_concurrent_streams(cuda):
    # long-K GEMMs with many tile rounds run with the round-synchronised
    # producers (a per-stream arrival counter): two of them concurrently on
    # two streams must give exactly their single-stream results
    g = torch.Generator(device="cuda").manual_seed(23)
    a = [((torch.rand(8192, 4096, generator=g, device="cuda") - 0.5)).bfloat16() for _ in range(2)]
    b = [((torch.rand(4096, 8192, generator=g, device="cuda") - 0.5) * 0.05).bfloat16() for _ in range(2)]
    bias = torch.rand(8192, generator=g, device="cuda")
    want = [ops.gemm(x, y, bias=bias, epilogue=Epilogue.BIAS_GELU_TANH) for x, y in zip(a, b)]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for _ in range(3):
        got = []
        for s, x, y in zip(streams, a, b):
            with torch.cuda.stream(s):
                got.append(ops.gemm(x, y, bias=bias, epilogue=Epilogue.BIAS_GELU_TANH))
        torch.cuda.synchronize()
        for u, v in zip(got, want):
            assert torch.equal(u, v)
