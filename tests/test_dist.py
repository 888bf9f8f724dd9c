"""Multi-rank host logic of the sharded validator (paper_2410_23661_b200.dist),
world_size 2 on CPU with gloo: shard ranges, the all-gather of bit-packed
flags and the all-reduce of verdict counts.  The per-shard flags come from the
oracle here (the GPU path is covered by the -m gpu tests)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle.picker_oracle as O
from tracegen.synth import random_records, random_summary

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_ranges():
    from paper_2410_23661_b200.dist import padded_words, shard_range
    for n in [0, 1, 31, 32, 33, 1000, 12345, 1 << 20]:
        for world in [1, 2, 3, 4, 8]:
            rs = [shard_range(n, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            for (a, b), (c, d) in zip(rs, rs[1:]):
                assert b == c
            for a, b in rs:
                assert (a % 32 == 0 or a == b == n) and a <= b
                assert (b - a + 31) // 32 <= padded_words(n, world)


def _pack(codes):
    idem = (np.asarray(codes) <= 1).astype(np.uint8)
    n = len(idem)
    b = np.packbits(np.pad(idem, (0, (-n) % 32)).reshape(-1, 32)[:, ::-1], axis=1)
    return b.view(">u4").reshape(-1).astype(np.uint32).view(np.int32)


def _worker(rank, world, port, n, codes, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2410_23661_b200.dist import gather_bits, reduce_counts, shard_range
    lo, hi = shard_range(n, world, rank)
    local = torch.from_numpy(_pack(codes[lo:hi]).copy())
    full = gather_bits(local, n)
    cnt = torch.zeros(16, dtype=torch.int64)
    for c in codes[lo:hi]:
        cnt[c if c <= 11 else 15] += 1
    reduce_counts(cnt)
    out_q.put((rank, full.numpy().copy(), cnt.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gather_flags_and_counts(world):
    s = random_summary(77, n_kernels=10)
    rec, args = random_records(78, s, 1000 + 17, max_threads=16, max_grid=2)
    codes = np.array(O.oracle_batch(s, rec, args), np.uint8)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, len(codes), codes, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_bits = _pack(codes)
    want_cnt = np.zeros(16, np.int64)
    for c in codes:
        want_cnt[c if c <= 11 else 15] += 1
    for rank, bits, cnt in res:
        assert np.array_equal(bits, want_bits), rank
        assert np.array_equal(cnt, want_cnt), rank


# ---- the bench's N > 1 code path and the chunked exchange (gloo, CPU) ----------

class _OraclePicker:
    """Stands in for the GPU validator on CPU: flags / bits / counts of the
    oracle codes of the records it is given (same output contract)."""

    def __init__(self, summary, args):
        self.K = O.index_summary(summary)
        self.args = args

    def validate(self, rec, args, out=None, stream=None):
        codes = np.array([O.oracle_interval(self.K, O.decode_record(r, self.args)) for r in rec], np.uint8)
        flags, bits, counts = out
        flags.copy_(torch.from_numpy(codes))
        bits.copy_(torch.from_numpy(_pack(codes)))
        cnt = np.zeros(16, np.int64)
        for c in codes:
            cnt[c if c <= 11 else 15] += 1
        counts.copy_(torch.from_numpy(cnt))
        return flags, bits, counts


def _bench_worker(rank, world, port, nchunks, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2410_23661_b200 import dist as pdist
    from tracegen.workloads import replicate
    s = random_summary(91, n_kernels=12)
    base, args = random_records(92, s, 200 + 24, max_threads=16, max_grid=2)  # 224: whole words
    ptr = np.zeros(len(args), bool)
    # this rank's replicas (the bench's shard layout: R copies per rank)
    R = 3
    rec, a = replicate(base, args, ptr, R * world, delta=0)
    rec = rec[rank * R * len(base):(rank + 1) * R * len(base)]
    picker = _OraclePicker(s, a)
    n = len(rec)
    # (1) the bench's step: one validate of the whole shard, gather_bits_equal, reduce_counts
    flags = torch.empty(n, dtype=torch.uint8)
    bits = torch.empty((n + 31) // 32, dtype=torch.int32)
    counts = torch.empty(16, dtype=torch.int64)
    picker.validate(rec, a, out=(flags, bits, counts))
    g1 = pdist.gather_bits_equal(bits.clone())
    c1 = pdist.reduce_counts(counts.clone())
    # (2) validate_sharded over the unequal-shard helper (the whole stream sharded)
    full, _ = replicate(base, args, ptr, R * world, delta=0)
    lo, hi = pdist.shard_range(len(full), world, rank)

    class _P:
        def validate(self, r, a_, stream=None):
            f = torch.empty(len(r), dtype=torch.uint8)
            b = torch.empty((len(r) + 31) // 32, dtype=torch.int32)
            c = torch.empty(16, dtype=torch.int64)
            return picker.validate(r, a_, out=(f, b, c))

    _, g2, c2 = pdist.validate_sharded(_P(), full[lo:hi], a, len(full))
    # (3) the chunked, overlapped exchange
    ex = pdist.ChunkedExchange(picker, n, nchunks, "cpu")
    _, g3, c3 = ex.run(rec, a, validate=lambda r, out: picker.validate(r, a, out=out))
    out_q.put((rank, g1.numpy().copy(), c1.numpy().copy(), g2.numpy().copy(), c2.numpy().copy(),
               g3.numpy().copy(), c3.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,nchunks", [(2, 1), (2, 3), (3, 4)])
def test_bench_exchange_paths(world, nchunks):
    """The exact N > 1 calls of bench.py (gather_bits_equal + reduce_counts),
    validate_sharded and the chunked exchange all give every rank the global
    mask and histogram that one process computes over the same stream (P = 1),
    bit for bit ("gathered masks are bit-identical across P")."""
    from tracegen.workloads import replicate
    s = random_summary(91, n_kernels=12)
    base, args = random_records(92, s, 224, max_threads=16, max_grid=2)
    full, a = replicate(base, args, np.zeros(len(args), bool), 3 * world, delta=0)
    codes = np.array(O.oracle_batch(s, full, a), np.uint8)
    want_bits = _pack(codes)
    want_cnt = np.bincount(np.where(codes <= 11, codes, 15), minlength=16)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, nchunks, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, g1, c1, g2, c2, g3, c3 in res:
        for g, c in [(g1, c1), (g2, c2), (g3, c3)]:
            assert np.array_equal(g, want_bits), rank
            assert np.array_equal(c, want_cnt), rank
