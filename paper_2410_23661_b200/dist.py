"""Multi-GPU sharding of a launch-record stream (SURVEY §8 row e).

Records are independent (each instance is validated alone),
so the stream shards by instance with no data-path collective.  The one
exchange step is the north star's: every rank ends with every flag, via an
all-gather of the bit-packed idempotent masks (n/8 bytes in total) and an
all-reduce of the 16-bin verdict histogram, over NCCL (NVLink/NVSwitch) on GPU
or gloo on CPU (tests).

Shards are contiguous and sized in multiples of 32 records so that no ballot
word straddles two ranks; the last rank takes the remainder.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, world: int, rank: int):
    """[lo, hi) of rank's shard: 32-record aligned, balanced, covering [0, n)."""
    words = (n + 31) // 32
    per = words // world
    extra = words % world
    w_lo = rank * per + min(rank, extra)
    w_hi = w_lo + per + (1 if rank < extra else 0)
    return min(n, 32 * w_lo), min(n, 32 * w_hi)


def padded_words(n: int, world: int) -> int:
    """Words per rank in the all-gather buffer (max shard size, equal for all)."""
    words = (n + 31) // 32
    return (words + world - 1) // world


def gather_bits(local_bits: torch.Tensor, n: int, group=None) -> torch.Tensor:
    """All-gather each rank's idempotent-bit words into the full mask of n records."""
    world = dist.get_world_size(group)
    pw = padded_words(n, world)
    buf = torch.zeros(pw, dtype=torch.int32, device=local_bits.device)
    buf[: local_bits.numel()] = local_bits
    out = torch.empty(pw * world, dtype=torch.int32, device=local_bits.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    # drop each rank's padding: rank r's words start at its shard's first word
    parts = []
    for r in range(world):
        lo, hi = shard_range(n, world, r)
        nw = (hi - lo + 31) // 32
        parts.append(out[r * pw: r * pw + nw])
    return torch.cat(parts)


def gather_bits_equal(local_bits: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather when every rank holds a shard of the same size (rank-major
    result; each rank's mask ends on a word boundary, its pad bits are 0)."""
    world = dist.get_world_size(group)
    out = torch.empty(local_bits.numel() * world, dtype=local_bits.dtype, device=local_bits.device)
    dist.all_gather_into_tensor(out, local_bits, group=group)
    return out


def reduce_counts(counts: torch.Tensor, group=None) -> torch.Tensor:
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def validate_sharded(picker, rec_shard, args_shard, n_total: int, *, stream=None, group=None):
    """Validate this rank's shard on its GPU, then exchange flags and counts.

    Returns (local flags u8, global bits i32[ceil(n_total/32)], global counts i64[16])."""
    flags, bits, counts = picker.validate(rec_shard, args_shard, stream=stream)
    gbits = gather_bits(bits, n_total, group)
    gcounts = reduce_counts(counts, group)
    return flags, gbits, gcounts
