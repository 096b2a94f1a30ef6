"""GPU parity of K1c (int8 GEMM, tcgen05 kind::i8; the quant module's
repositioned matmul) against the integer oracle
(oracle.matmul_i8) and the reference interpreter's own outputs
(tests/golden/int8_matmul.json). Integer work: bit-exact, tolerance 0 —
including the requantised i8 (round half away from zero, saturating) and the
dequantised f32 (acc * scale in double, rounded once to f32)."""
import json
import os

import numpy as np
import pytest
import torch

import oracle as O
from paper_2603_06731_b200 import AfgError, ops

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def i8(shape, seed):
    g = torch.Generator().manual_seed(seed)
    return torch.randint(-128, 128, shape, generator=g, dtype=torch.int8)


def test_reference_fixtures_bit_exact(cuda):
    for c in json.load(open(os.path.join(GOLD, "int8_matmul.json")))["cases"]:
        a = np.array(c["a"], dtype=np.int8)
        b = np.array(c["b"], dtype=np.int8)
        K = a.shape[1]
        Kp = (K + 15) // 16 * 16  # TMA row pitch: 16 bytes
        ad = torch.zeros((a.shape[0], Kp), dtype=torch.int8)
        ad[:, :K] = torch.from_numpy(a)
        bd = torch.zeros((b.shape[1], Kp), dtype=torch.int8)
        bd[:, :K] = torch.from_numpy(np.ascontiguousarray(b.T))
        got = ops.gemm_i8(ad.cuda()[:, :K], bd.cuda()[:, :K]).cpu().numpy()
        assert np.array_equal(got, np.array(c["c"])), c["name"]


@pytest.mark.parametrize("M,N,K", [(128, 256, 128), (333, 200, 144), (1000, 520, 1040),
                                   (64, 64, 16), (2048, 1024, 4096)])
def test_i32_exact(cuda, M, N, K):
    a, b = i8((M, K), M), i8((N, K), N + 1)
    got = ops.gemm_i8(a.cuda(), b.cuda()).cpu().numpy()
    rows = None if M * N * K <= 2**28 else np.r_[0:3, M // 2, M - 1]
    want = O.matmul_i8(a.numpy(), b.numpy(), rows=rows)
    assert np.array_equal(got if rows is None else got[rows], want)


@pytest.mark.parametrize("mode,scale", [(1, 1 / 4096), (1, 0.5), (2, 3.1e-5), (1, 1 / 1000.3),
                                        (1, 0.013), (2, 0.1)])
def test_requant_and_dequant(cuda, mode, scale):
    M, N, K = 300, 384, 512
    a, b = i8((M, K), 5), i8((N, K), 6)
    got = ops.gemm_i8(a.cuda(), b.cuda(), out_mode=mode, scale=scale).cpu().numpy()
    want = O.matmul_i8(a.numpy(), b.numpy(), mode=mode, scale=scale)
    assert np.array_equal(got, want)
    if mode == 1 and scale == 0.5:  # saturates both ways
        assert (got == 127).any() and (got == -128).any()


def test_many_tiles_per_cta(cuda):
    """>= 3 tiles per persistent CTA (TMEM accumulator double-buffer phases)."""
    M, N, K = 148 * 128 * 3 + 50, 256, 256
    a, b = i8((M, K), 9), i8((N, K), 10)
    got = ops.gemm_i8(a.cuda(), b.cuda()).cpu().numpy()
    rows = np.arange(0, M, 997)
    assert np.array_equal(got[rows], O.matmul_i8(a.numpy(), b.numpy(), rows=rows))


def test_rejects_unaligned_pitch(cuda):
    a = torch.zeros((8, 20), dtype=torch.int8, device="cuda")
    b = torch.zeros((8, 20), dtype=torch.int8, device="cuda")
    with pytest.raises(AfgError):
        ops.gemm_i8(a, b)


# 256 x 256 tiles on a CTA pair (cta_group::2 kind::i8) once there are >= 74 of
# them: ragged M / N / K, every output mode, and >= 3 pair tiles per cluster.
@pytest.mark.parametrize("mode,scale", [(0, 1.0), (1, 1 / 2048), (2, 1e-3)])
def test_pair_tiles_ragged(cuda, mode, scale):
    M, N, K = 2500, 2000, 208
    a, b = i8((M, K), 11), i8((N, K), 12)
    got = ops.gemm_i8(a.cuda(), b.cuda(), out_mode=mode, scale=scale).cpu().numpy()
    rows = np.r_[0:2, 127:130, 255:258, 1024, 2047, 2300, M - 1]
    assert np.array_equal(got[rows], O.matmul_i8(a.numpy(), b.numpy(), mode=mode, scale=scale,
                                                 rows=rows))


def test_pair_tiles_long_k_many_per_cluster(cuda):
    M, N, K = 256 * 74 * 3 + 100, 512, 1024
    a, b = i8((M, K), 13), i8((N, K), 14)
    got = ops.gemm_i8(a.cuda(), b.cuda()).cpu().numpy()
    rows = np.arange(0, M, 1009)
    assert np.array_equal(got[rows], O.matmul_i8(a.numpy(), b.numpy(), rows=rows))


@pytest.mark.parametrize("mode,scale", [(1, 1 / 140000.7), (2, 1e-3)])
def test_large_accumulators_take_the_double_path(cuda, mode, scale):
    """|acc| >= 2^24 (float no longer exact): the epilogue's double fallback."""
    M, N, K = 128, 256, 1088
    a = torch.full((M, K), 127, dtype=torch.int8)
    a[1::2] = -127
    b = torch.full((N, K), 127, dtype=torch.int8)
    b[:, ::3] = 126
    got = ops.gemm_i8(a.cuda(), b.cuda(), out_mode=mode, scale=scale).cpu().numpy()
    want = O.matmul_i8(a.numpy(), b.numpy(), mode=mode, scale=scale)
    assert np.abs(O.matmul_i8(a.numpy(), b.numpy())).min() >= 2**24
    assert np.array_equal(got, want)


# ------------------------------------------------ int8 implicit-GEMM conv ---

def test_conv_reference_fixtures_bit_exact(cuda):
    for c in json.load(open(os.path.join(GOLD, "int8_matmul.json")))["conv_cases"]:
        x = torch.from_numpy(np.ascontiguousarray(np.transpose(np.array(c["x"], dtype=np.int8),
                                                               (0, 2, 3, 1))))
        w = torch.from_numpy(np.ascontiguousarray(np.transpose(np.array(c["w"], dtype=np.int8),
                                                               (0, 2, 3, 1))))
        K = w.shape[1]
        y = np.array(c["y"])
        pad = (K // 2, K // 2) if c["padding"] == "same" else (0, 0)
        got = ops.conv2d_nhwc_i8(x.cuda(), w.cuda(), stride=(c["stride"],) * 2, pad=pad,
                                 out_hw=(y.shape[2], y.shape[3])).cpu().numpy()
        assert np.array_equal(np.transpose(got, (0, 3, 1, 2)), y), c["name"]


@pytest.mark.parametrize("B,H,C,OC,K,s,p", [(4, 28, 128, 128, 3, 1, 1), (2, 56, 64, 96, 3, 2, 1),
                                            (4, 14, 256, 64, 1, 1, 0), (3, 13, 48, 40, 3, 1, 1),
                                            (2, 7, 512, 300, 3, 1, 1)])
def test_conv_shapes_i32_exact(cuda, B, H, C, OC, K, s, p):
    x, w = i8((B, H, H, C), H + C), i8((OC, K, K, C), OC + K)
    got = ops.conv2d_nhwc_i8(x.cuda(), w.cuda(), stride=(s, s), pad=(p, p)).cpu().numpy()
    want = O.conv_i8(x.numpy(), w.numpy(), stride=(s, s), pad=(p, p))
    assert np.array_equal(got, want)


@pytest.mark.parametrize("mode,scale", [(1, 1 / 3000.7), (2, 1e-3)])
def test_conv_requant_and_dequant(cuda, mode, scale):
    x, w = i8((2, 20, 20, 64), 31), i8((128, 3, 3, 64), 32)
    got = ops.conv2d_nhwc_i8(x.cuda(), w.cuda(), pad=(1, 1), out_mode=mode, scale=scale)
    want = O.conv_i8(x.numpy(), w.numpy(), pad=(1, 1), mode=mode, scale=scale)
    assert np.array_equal(got.cpu().numpy(), want)
