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
