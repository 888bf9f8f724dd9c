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


class ChunkedExchange:
    """Validation of a rank's shard in chunks, each chunk's flag-bit all-gather
    overlapped with the next chunk's validation (SURVEY §8 row e: "chunked
    overlap on a second stream hides the rest").

    Every rank holds a shard of the same number of records, split into
    `nchunks` chunks of whole 32-record words.  Chunk c is validated on the
    compute stream; an event marks its end; the communication stream waits for
    it and all-gathers the chunk's bit words into their final place in the
    global mask (rank-major: rank r's shard is records [r*n_local, (r+1)*n_local)),
    while chunk c+1 is already validating.  The counts are all-reduced once.
    On CPU (gloo) the streams are absent and the same calls run in order.
    """

    def __init__(self, picker, n_local: int, nchunks: int, device, group=None):
        self.p = picker
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n_local = n_local
        self.words = (n_local + 31) // 32
        per = (self.words + nchunks - 1) // max(nchunks, 1)
        self.bounds = [(w * 32, min(n_local, (w + per) * 32)) for w in range(0, self.words, per)] or [(0, 0)]
        self.device = torch.device(device)
        cuda = self.device.type == "cuda"
        self.comm = torch.cuda.Stream(self.device) if cuda else None
        self.flags = torch.empty(n_local, dtype=torch.uint8, device=self.device)
        self.bits = torch.empty(self.words, dtype=torch.int32, device=self.device)
        self.counts = torch.empty(16, dtype=torch.int64, device=self.device)
        self.chunk_counts = torch.empty(len(self.bounds), 16, dtype=torch.int64, device=self.device)
        self.gbits = torch.empty(self.world * self.words, dtype=torch.int32, device=self.device)

    def _views(self, c):
        lo, hi = self.bounds[c]
        w0, w1 = lo // 32, (hi + 31) // 32
        return [self.gbits[r * self.words + w0: r * self.words + w1] for r in range(self.world)]

    def run(self, rec, args, *, validate=None):
        """Validate `rec` (this rank's shard, device records) chunk by chunk and
        exchange.  Returns (local flags, global bits i32[world * words], global
        counts i64[16]); all valid on the current stream after the call.
        `validate(rec_chunk, out)` overrides the picker call (tests)."""
        cur = torch.cuda.current_stream(self.device) if self.comm is not None else None
        works = []
        for c, (lo, hi) in enumerate(self.bounds):
            out = (self.flags[lo:hi], self.bits[lo // 32:(hi + 31) // 32], self.chunk_counts[c])
            if validate is None:
                self.p.validate(rec[lo:hi], args, out=out, stream=cur)
            else:
                validate(rec[lo:hi], out)
            if self.comm is not None:
                ev = torch.cuda.Event()
                ev.record(cur)
                self.comm.wait_event(ev)
                with torch.cuda.stream(self.comm):
                    works.append(dist.all_gather(self._views(c), out[1], group=self.group, async_op=True))
            else:
                dist.all_gather(self._views(c), out[1], group=self.group)
        for w in works:
            w.wait()
        if self.comm is not None:
            cur.wait_stream(self.comm)
        torch.sum(self.chunk_counts, dim=0, out=self.counts)
        dist.all_reduce(self.counts, op=dist.ReduceOp.SUM, group=self.group)
        return self.flags, self.gbits, self.counts
