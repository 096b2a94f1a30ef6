"""Split-K / tensor-parallel GEMM (north-star item 4): the one
BASELINE path with a real exchange step, as a binding of the C ABI
(afg_gemm_splitk, csrc/tp.cpp).

Rank r of P holds the K slice A[:, K_r] and B[K_r, :] (the row-parallel linear
layer layout). afg_gemm_splitk computes the rank's fp32 partial on the
tensor cores, sums the partials across ranks with NCCL over NVLink
(reduce-scatter into row blocks, or all-reduce), and applies the bias /
activation epilogue to the sum. Communicators come from the C ABI
(afg_comm_*): per rank from a unique id shared through the job's
torch.distributed group, or for all local devices of a thread-per-device
group (afg_group_*, include/afg_multi.h).
"""
from __future__ import annotations

import ctypes

import torch

from . import Epilogue, check, lib
from .ops import _need_cuda, _ptr, _stream, afg_dtype
from .shard import shard_rows

REDUCE_SCATTER = 0
ALL_REDUCE = 1


def split_plan(M: int, K: int, rank: int, world: int, mode: int = REDUCE_SCATTER):
    """(k0, k1) of this rank's K slice and (r0, r1) of the output rows it
    owns after the exchange (all rows for ALL_REDUCE)."""
    k0, k1 = shard_rows(K, rank, world)
    if mode == REDUCE_SCATTER:
        if M % world:
            raise ValueError(f"reduce-scatter needs M % world == 0 (M={M}, world={world})")
        rows = M // world
        return (k0, k1), (rank * rows, (rank + 1) * rows)
    return (k0, k1), (0, M)


class Comm:
    """An NCCL communicator owned by afg (ncclComm_t)."""

    def __init__(self, handle: int, rank: int, world: int):
        self.handle, self.rank, self.world = handle, rank, world

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        check(lib().afg_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def from_unique_id(cls, uid: bytes, rank: int, world: int) -> "Comm":
        h = ctypes.c_void_p()
        check(lib().afg_comm_init_rank(ctypes.byref(h), world, ctypes.c_char_p(uid), rank))
        return cls(h.value, rank, world)

    @classmethod
    def from_process_group(cls, group=None) -> "Comm":
        """One communicator per rank of the torch.distributed job: rank 0
        creates the unique id, the group broadcasts it."""
        import torch.distributed as dist
        if not dist.is_available() or not dist.is_initialized():
            return cls.from_unique_id(cls.unique_id(), 0, 1)
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        box = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=group)
        return cls.from_unique_id(box[0], rank, world)

    @staticmethod
    def for_devices(devices) -> list["Comm"]:
        n = len(devices)
        hs = (ctypes.c_void_p * n)()
        devs = (ctypes.c_int * n)(*devices)
        check(lib().afg_comm_init_all(hs, n, devs))
        return [Comm(hs[i], i, n) for i in range(n)]

    def close(self):
        if self.handle:
            lib().afg_comm_destroy(ctypes.c_void_p(self.handle))
            self.handle = None


def gemm_splitk(a_k: torch.Tensor, b_k: torch.Tensor, comm: Comm, bias=None,
                epilogue: Epilogue = Epilogue.NONE, out_dtype=torch.bfloat16,
                mode: int = REDUCE_SCATTER, out=None, workspace=None) -> torch.Tensor:
    """epi(sum over ranks of a_k @ b_k + bias): this rank's row block
    ([M/P, N], REDUCE_SCATTER) or the full [M, N] (ALL_REDUCE)."""
    _need_cuda(a_k, b_k, bias, out)
    M, K_local = a_k.shape
    N = b_k.shape[1]
    rows = M // comm.world if mode == REDUCE_SCATTER else M
    if out is None:
        out = torch.empty((rows, N), dtype=out_dtype, device=a_k.device)
    L = lib()
    ws_bytes = L.afg_gemm_splitk_workspace(M, N, comm.world, mode)
    if workspace is None or workspace.numel() < ws_bytes:
        workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=a_k.device)
    check(L.afg_gemm_splitk(_ptr(a_k), a_k.stride(0), _ptr(b_k), b_k.stride(0), _ptr(bias),
                            _ptr(out), out.stride(0), M, N, K_local, afg_dtype(a_k.dtype),
                            afg_dtype(out.dtype), 0, int(epilogue), ctypes.c_void_p(comm.handle),
                            mode, _ptr(workspace), ws_bytes, _stream()))
    return out
