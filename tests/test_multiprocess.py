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
    """Host side of the split-K path on gloo: the K slices / output row blocks
    of split_plan, and the NCCL unique-id handshake Comm.from_process_group
    performs (rank 0's afg_comm_unique_id bytes broadcast to every rank)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_06731_b200 import AfgError
        from paper_2603_06731_b200.tp import ALL_REDUCE, REDUCE_SCATTER, Comm, split_plan
        plans = [split_plan(36, 64, rank, world, m) for m in (REDUCE_SCATTER, ALL_REDUCE)]
        try:
            uid = Comm.unique_id() if rank == 0 else None
        except AfgError as e:  # no libnccl / no network interface: handshake untestable here
            uid = ("unavailable", str(e))
        box = [uid]
        dist.broadcast_object_list(box, src=0)
        got = [None] * world
        dist.all_gather_object(got, (plans, box[0]))
        if rank == 0:
            q.put(got)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_splitk_plan_and_id_handshake():
    world, port = 2, free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_splitk_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (rs0, ar0), uid0 = got[0]
    (rs1, ar1), uid1 = got[1]
    # K slices tile [0, K) without overlap; reduce-scatter rows tile [0, M)
    assert rs0[0] == (0, 32) and rs1[0] == (32, 64)
    assert rs0[1] == (0, 18) and rs1[1] == (18, 36)
    assert ar0[1] == ar1[1] == (0, 36)
    assert uid0 == uid1  # every rank sees rank 0's id
    if not (isinstance(uid0, tuple) and uid0[0] == "unavailable"):
        assert isinstance(uid0, bytes) and len(uid0) == 128 and any(uid0)
