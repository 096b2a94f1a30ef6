"""CPU tests of the N>1 host path (gloo, world_size 2, 127.0.0.1): the row /
head / batch sharding plans of paper_2603_06731_b200.shard, the sharded
synthetic-input streams, and the max-over-ranks timing reduction that
bench.py uses under torchrun. Each rank computes its shard of the GEMM with
the oracle; the gathered shards must equal the single-process result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2603_06731_b200.shard import max_over_ranks, shard_rows, shard_seed


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_rows_cover_exactly():
    for total in (1, 7, 128, 16384, 16385):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_rows(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_rows(10, 2, 2)


def test_shard_seed_streams_concatenate():
    s0 = O.stream_seed("%a", 1)
    full = O.random_stream((64, 48), s0, -1, 1)
    parts = []
    for r in range(3):
        a, b = shard_rows(64, r, 3)
        parts.append(O.random_stream((b - a, 48), shard_seed(s0, a * 48), -1, 1))
    assert np.array_equal(np.concatenate(parts), full)
    # and the unsharded stream is the reference generator's
    assert np.array_equal(full, O.random_tensor((64, 48), "%a", 1, -1, 1))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        M, K, N = 40, 24, 16
        a0, a1 = shard_rows(M, rank, world)
        sa = O.stream_seed("%a", 5)
        A = O.random_stream((a1 - a0, K), shard_seed(sa, a0 * K), -1, 1)
        B = O.random_stream((K, N), O.stream_seed("%b", 5), -1, 1)
        C = O.matmul(O.round_to(A, O.F32), O.round_to(B, O.F32), interp=True)
        shards = [None] * world
        dist.all_gather_object(shards, C)
        t = max_over_ranks(float(rank + 1))
        # head sharding of an attention batch: (b, h) pairs
        h0, h1 = shard_rows(8 * 16, rank, world)
        heads = list(range(h0, h1))
        all_heads = [None] * world
        dist.all_gather_object(all_heads, heads)
        if rank == 0:
            q.put((np.concatenate(shards), t, sum(all_heads, [])))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_row_sharded_gemm_and_timing():
    world, port = 2, free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    C, t, heads = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    M, K, N = 40, 24, 16
    A = O.random_tensor((M, K), "%a", 5, -1, 1)
    B = O.random_tensor((K, N), "%b", 5, -1, 1)
    want = O.matmul(O.round_to(A, O.F32), O.round_to(B, O.F32), interp=True)
    assert np.array_equal(C, want)
    assert t == 2.0  # max over ranks
    assert heads == list(range(128))


def _splitk_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_06731_b200.tp import gemm_splitk
        M, K, N = 36, 64, 20
        A = O.random_tensor((M, K), "%a", 7, -1, 1)
        B = O.random_tensor((K, N), "%b", 7, -1, 1)
        k0, k1 = shard_rows(K, rank, world)
        fn = lambda a, b: torch.from_numpy(O.matmul(a.numpy(), b.numpy()))  # noqa: E731
        shard = gemm_splitk(torch.from_numpy(A[:, k0:k1].copy()),
                            torch.from_numpy(B[k0:k1].copy()), partial_fn=fn)
        out = [None] * world
        dist.all_gather_object(out, shard.numpy())
        if rank == 0:
            q.put(np.concatenate(out))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_splitk_reduce_scatter():
    world, port = 2, free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_splitk_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    C = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = O.random_tensor((36, 64), "%a", 7, -1, 1)
    B = O.random_tensor((64, 20), "%b", 7, -1, 1)
    # sum of two f32-rounded half-K partials vs the full product
    ok, ma, mr, _ = O.compare(C, O.matmul(A, B), 1e-6)
    assert ok, mr
