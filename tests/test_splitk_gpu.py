"""Split-K / tensor-parallel GEMM through the C ABI (afg_gemm_splitk:
tcgen05 fp32 partial -> NCCL reduce-scatter / all-reduce -> epilogue) and the
thread-per-device group (afg_group_*), on the GPUs of this box.

One GPU: a one-rank communicator (from a unique id, and from
ncclCommInitAll) -- the exchange is then the identity and the result must be
the oracle's epi(A B + bias). Two or more GPUs: a 2-process job with the
K dimension split, the row blocks gathered and checked against the full
product (skipped when fewer than two GPUs are visible).

Tolerance: bf16 output, one bf16 ulp of the double oracle on the same
bf16 inputs (2^-7 relative, the SURVEY §8c bf16 rule); fp32 output 1e-5."""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch

import oracle as O
from paper_2603_06731_b200 import Epilogue, check, lib
from paper_2603_06731_b200.tp import ALL_REDUCE, REDUCE_SCATTER, Comm, gemm_splitk, split_plan
from tests.gpu_util import seeded, to_host

pytestmark = pytest.mark.gpu


def _operands(M, N, K, seed=5):
    a, ah = seeded((M, K), "a", seed)
    b, bh = seeded((K, N), "b", seed)
    bias, biash = seeded((N,), "bias", seed, dtype=torch.float32)
    return a, ah, b, bh, bias, biash


@pytest.mark.parametrize("mode", [REDUCE_SCATTER, ALL_REDUCE])
@pytest.mark.parametrize("how", ["unique_id", "init_all"])
def test_splitk_one_rank(cuda, mode, how):
    M, N, K = 256, 384, 512
    a, ah, b, bh, bias, biash = _operands(M, N, K)
    comm = Comm.from_unique_id(Comm.unique_id(), 0, 1) if how == "unique_id" else \
        Comm.for_devices([0])[0]
    try:
        out = gemm_splitk(a, b, comm, bias=bias, epilogue=Epilogue.BIAS_GELU_TANH,
                          out_dtype=torch.float32, mode=mode)
        torch.cuda.synchronize()
    finally:
        comm.close()
    want = O.matmul(ah, bh, biash, epi=O.EPI_GELU_TANH, out_t=O.F64)
    ok, ma, mr, w = O.compare(to_host(out), want, 1e-5)
    assert ok, f"max_rel {mr:.3e} at {w}"


def test_device_group_runs_on_its_thread_and_stream(cuda):
    """afg_group_run: the callback runs on the device's worker thread with the
    group's stream; an afg_gemm issued there matches the oracle."""
    L = lib()
    M, N, K = 128, 256, 192
    a, ah, b, bh, bias, biash = _operands(M, N, K, seed=9)
    c = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    torch.cuda.synchronize()
    seen = []
    FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                          ctypes.c_void_p, ctypes.c_void_p)

    def job(user, rank, device, stream, comm):
        seen.append((rank, device, bool(stream), comm))
        return L.afg_gemm(a.data_ptr(), K, b.data_ptr(), N, bias.data_ptr(), None, c.data_ptr(),
                          N, M, N, K, 2, 2, 0, int(Epilogue.BIAS_RELU), ctypes.c_void_p(stream))

    cb = FN(job)
    g = ctypes.c_void_p()
    devs = (ctypes.c_int * 1)(0)
    check(L.afg_group_create(1, devs, ctypes.byref(g)))
    try:
        assert L.afg_group_size(g) == 1
        check(L.afg_group_run(g, ctypes.cast(cb, ctypes.c_void_p), None))
    finally:
        L.afg_group_destroy(g)
    assert seen == [(0, 0, True, None)]
    want = O.round_to(O.matmul(ah, bh, biash, epi=O.EPI_RELU, out_t=O.F64), O.BF16)
    ok, ma, mr, w = O.compare(to_host(c), want, 2.0 ** -7)
    assert ok, mr


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    M, N, K = 256, 384, 1024
    A = O.round_to(O.random_tensor((M, K), "%a", 3, -1, 1), O.BF16)
    B = O.round_to(O.random_tensor((K, N), "%b", 3, -1, 1), O.BF16)
    (k0, k1), (r0, r1) = split_plan(M, K, rank, world)
    a = torch.from_numpy(A[:, k0:k1].copy()).to(torch.bfloat16).cuda()
    b = torch.from_numpy(B[k0:k1].copy()).to(torch.bfloat16).cuda()
    comm = Comm.from_process_group()
    out = gemm_splitk(a, b, comm, out_dtype=torch.float32)
    torch.cuda.synchronize()
    got = [None] * world
    dist.all_gather_object(got, out.cpu().double().numpy())
    if rank == 0:
        q.put(np.concatenate(got))
    comm.close()
    dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_splitk_two_ranks_nccl():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    C = q.get(timeout=300)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    A = O.round_to(O.random_tensor((256, 1024), "%a", 3, -1, 1), O.BF16)
    B = O.round_to(O.random_tensor((1024, 384), "%b", 3, -1, 1), O.BF16)
    ok, ma, mr, w = O.compare(C, O.matmul(A, B, out_t=O.F64), 1e-5)
    assert ok, mr
