"""Multi-GPU sharding plans: one process per GPU, every
BASELINE config partitions with no data-path collective.

  gemm (configs[1])      rows of A / C, B replicated          shard_rows(M)
  attention (configs[2]) flattened (b, h) pairs               shard_rows(B*H)
  ResNet convs / BERT    batch                                shard_rows(B)
  softmax / layernorm    rows                                 shard_rows(rows)
  fp32 1024^3 (configs[0]) replicas (too small to split)

Synthetic inputs are generated on the device from the reference's
makeRandomTensor stream (interp.cpp:817-844); shard_seed() offsets the stream
so that the concatenation of the rank shards is bit-identical to the
single-GPU tensor."""
from __future__ import annotations

GOLDEN = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1


def shard_rows(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [begin, end) shard of `total` units for `rank` (remainder
    spread over the first ranks)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(total, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def shard_seed(s0: int, first_element: int) -> int:
    """Stream state whose draw i equals draw (first_element + i) of stream s0:
    splitmix64 advances its state by the golden constant per draw."""
    return (s0 + first_element * GOLDEN) & MASK64


def max_over_ranks(value: float, group=None) -> float:
    """Device time of a step = the slowest rank (all_reduce MAX)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
