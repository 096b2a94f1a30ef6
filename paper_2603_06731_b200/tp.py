"""Split-K / tensor-parallel GEMM (north-star item 4): the only
BASELINE path with a real exchange step.

Rank r holds the K-slice A[:, K_r] and B[K_r, :] (tensor-parallel layout of a
row-parallel linear layer). Each rank computes its fp32 partial
C_r = A[:, K_r] B[K_r, :] with the tcgen05 GEMM (afg_gemm, fp32 out, no
epilogue), the partials are summed with a reduce-scatter (NCCL over
NVLink/NVSwitch under torchrun) so rank r owns rows M_r of C, and the
bias + activation + convert epilogue is applied to that shard
(afg_epilogue_apply). The collective is a separate call today; fusing it
into the GEMM epilogue over peer memory / NVLS multicast is the next step.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import Epilogue, check, lib
from .ops import _ptr, _stream, afg_dtype, gemm
from .shard import shard_rows


def reduce_scatter_rows(partial: torch.Tensor, group=None) -> torch.Tensor:
    """Sum `partial` [M, N] over ranks; return this rank's row shard."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    M = partial.shape[0]
    if world == 1:
        return partial
    if M % world == 0 and dist.get_backend(group) == "nccl":
        out = torch.empty((M // world, partial.shape[1]), dtype=partial.dtype, device=partial.device)
        dist.reduce_scatter_tensor(out, partial, op=dist.ReduceOp.SUM, group=group)
        return out
    dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)
    r0, r1 = shard_rows(M, rank, world)
    return partial[r0:r1].contiguous()


def finish_epilogue(acc: torch.Tensor, bias, epilogue: Epilogue, out_dtype) -> torch.Tensor:
    out = torch.empty(acc.shape, dtype=out_dtype, device=acc.device)
    check(lib().afg_epilogue_apply(_ptr(acc), _ptr(bias), None, _ptr(out), acc.shape[0],
                                   acc.shape[1], acc.stride(0), int(epilogue),
                                   afg_dtype(acc.dtype), afg_dtype(out_dtype), _stream()))
    return out


def gemm_splitk(a_k: torch.Tensor, b_k: torch.Tensor, bias=None,
                epilogue: Epilogue = Epilogue.NONE, out_dtype=torch.bfloat16, group=None,
                partial_fn=None):
    """C[M_r, :] = epi(sum_r A[:, K_r] B[K_r, :] + bias) for this rank's rows.
    partial_fn (tests only) replaces the GPU partial GEMM."""
    if partial_fn is None:
        partial = gemm(a_k, b_k, out_dtype=torch.float32)
    else:
        partial = partial_fn(a_k, b_k)
    shard = reduce_scatter_rows(partial, group)
    if partial_fn is not None:
        return shard
    return finish_epilogue(shard, bias, epilogue, out_dtype)
