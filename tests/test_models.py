"""Row f3: consumer models on the verdicts (§7.5 l.1612-1690) --
Asymmetric-Resilience checkpoint bytes and Chimera preemption latency.

CPU pins: input bytes from the golden examples' hand-derived extents (the union
of read extents), the SPEC's model examples (all idempotent -> the kill latency;
half NI with equal sizes -> half the bytes; zero sizes -> zero), and the
4-98 us band of PAPER l.1683-1684.  GPU: picker_consumer_models against
oracle_models, integer-exact."""
import json
import os

import numpy as np
import pytest

import oracle.picker_oracle as O
from tracegen import golden
from tracegen.records import RecordBuilder
from tracegen.synth import random_records, random_summary

HERE = os.path.dirname(__file__)


def _rec(kid, args, grid=(1, 1, 1), block=(1, 1, 1)):
    b = RecordBuilder()
    b.add(kid, args, grid=grid, block=block)
    rec, pool = b.build()
    return O.decode_record(rec[0], pool)


@pytest.fixture(scope="module")
def G():
    return O.index_summary(golden.golden_summary())


def test_input_bytes_from_golden_extents(G):
    """Input bytes = total length of the union of the read extents the golden
    file lists (hand-derived from the cited passages)."""
    cases = json.load(open(os.path.join(HERE, "golden", "paper_examples.json")))["cases"]
    seen = 0
    for c in cases:
        if "extents" not in c:
            continue
        reads = sorted((lb, ub) for k, lb, ub in c["extents"] if k == "R")
        want = 0
        end = None
        for lb, ub in reads:  # the golden extents are disjoint or nested
            if end is None or lb > end:
                want += ub - lb + 1
                end = ub
            elif ub > end:
                want += ub - end
                end = ub
        r = _rec(c["kernel_id"], c["args"], c["grid"], c["block"])
        assert O.oracle_input_bytes(G, r) == want, c["name"]
        seen += 1
    assert seen >= 5


def test_input_bytes_union_not_sum(G):
    """vectorAdd (Fig. 1) reading B and C: 4 bytes per thread each; with C = B the
    checkpoint copies the one buffer once."""
    g, b = 4, 128
    assert O.oracle_input_bytes(G, _rec(0, [4096, 8192, 12288], (g, 1, 1), (b, 1, 1))) == 2 * 4 * g * b
    assert O.oracle_input_bytes(G, _rec(0, [4096, 8192, 8192], (g, 1, 1), (b, 1, 1))) == 4 * g * b


def test_input_bytes_classes(G):
    assert O.oracle_input_bytes(G, _rec(1, [4096], (4, 1, 1), (128, 1, 1))) == 0   # vectorSet: no reads
    assert O.oracle_input_bytes(G, _rec(2, [4096], (4, 1, 1), (128, 1, 1))) is None  # NONIDEM SO
    assert O.oracle_input_bytes(G, _rec(7, [4096, 8192, 1], (1, 1, 1), (32, 1, 1))) is None  # opaque read on


def _models_batch(codes_fn, ctx_fn, n=64):
    s = golden.golden_summary()
    b = RecordBuilder()
    for i in range(n):
        b.add(0, [4096 + (i << 20), 8192 + (i << 20), 12288 + (i << 20)], (4, 1, 1), (128, 1, 1))
    rec, args = b.build()
    codes = np.array([codes_fn(i) for i in range(n)], np.uint8)
    ctx = np.array([ctx_fn(i) for i in range(n)], np.uint64)
    return s, rec, args, codes, ctx


def test_models_all_idempotent():
    """SPEC: all instances idempotent -> AR copies nothing; mean preemption = kill."""
    s, rec, args, codes, ctx = _models_batch(lambda i: 0, lambda i: 50_000)
    m = O.oracle_models(s, rec, args, codes, ctx, kill_ns=1000, save_bytes_per_us=1000)
    assert m["ckpt_bytes_ni"] == 0 and m["ckpt_bytes_all"] == 64 * 4096
    assert m["preempt_ns_with"] == 64 * 1000 and m["preempt_ns_without"] == 64 * 50_000
    assert m["hist_with"][1] == 64


def test_models_half_ni_linear():
    """SPEC: half the instances NI with equal sizes -> half the checkpoint bytes."""
    s, rec, args, codes, ctx = _models_batch(lambda i: 10 if i % 2 else 0, lambda i: 0)
    m = O.oracle_models(s, rec, args, codes, ctx)
    assert 2 * m["ckpt_bytes_ni"] == m["ckpt_bytes_all"]
    assert m["preempt_ns_without"] == 0 and m["preempt_ns_with"] == 32 * 1000


def test_models_chimera_band():
    """without idempotency, latency 4-98 us depending on the
    context size; with contexts uniform in that band the mean lies in it."""
    rng = np.random.default_rng(3)
    sizes = rng.integers(4_000, 98_001, 64)
    s, rec, args, codes, ctx = _models_batch(lambda i: 10, lambda i: int(sizes[i]))
    m = O.oracle_models(s, rec, args, codes, ctx, save_bytes_per_us=1000)
    mean_us = m["preempt_ns_without"] / 64 / 1000
    assert 4 <= mean_us <= 98
    assert sum(m["hist_without"][4:99]) == 64


# ---- GPU parity ----------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("seed", [81, 82])
def test_gpu_models_random(seed):
    import paper_2410_23661_b200 as pk
    s = random_summary(seed, n_kernels=30)
    rec, args = random_records(seed + 1000, s, 3000, max_threads=256, max_grid=64)
    p = pk.Picker(0)
    p.load(s)
    flags, _, _ = p.validate(rec, args)
    codes = np.array(O.oracle_batch(s, rec, args), np.uint8)  # the oracle's verdicts, not the GPU's
    assert np.array_equal(flags.cpu().numpy(), codes)
    ctx = np.random.default_rng(seed).integers(0, 200_000, len(rec)).astype(np.uint64)
    got = p.consumer_models(rec, args, codes, ctx, kill_ns=1000, save_bytes_per_us=1500)
    want = O.oracle_models(s, rec, args, codes, ctx, kill_ns=1000, save_bytes_per_us=1500)
    assert got == want


@pytest.mark.gpu
def test_gpu_models_c2():
    import paper_2410_23661_b200 as pk
    from tracegen import workloads
    s, rec, args, _ = workloads.make_c2()
    p = pk.Picker(0)
    p.load(s)
    codes = np.array(O.oracle_batch_mp(s, rec, args), np.uint8)  # the oracle's verdicts
    ctx = np.random.default_rng(5).integers(4_000, 98_001, len(rec)).astype(np.uint64)
    got = p.consumer_models(rec, args, codes, ctx)
    want = O.oracle_models(s, rec, args, codes, ctx)
    assert got == want


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [81, 82])
def test_gpu_validate_models_random(seed):
    """Verdicts and models in one pass (picker_validate_models): the fused
    pipelined kernel for n > 1024, the two passes for a small batch; both equal
    to the oracle's verdicts and the oracle's models on them."""
    import paper_2410_23661_b200 as pk
    s = random_summary(seed, n_kernels=30)
    rec, args = random_records(seed + 1000, s, 3000, max_threads=256, max_grid=64)
    codes = np.array(O.oracle_batch(s, rec, args), np.uint8)
    ctx = np.random.default_rng(seed).integers(0, 200_000, len(rec)).astype(np.uint64)
    p = pk.Picker(0)
    p.load(s)
    for m in (len(rec), 700):
        (flags, bits, counts), got = p.validate_models(rec[:m], args, ctx[:m], kill_ns=1000, save_bytes_per_us=1500)
        assert np.array_equal(flags.cpu().numpy(), codes[:m])
        assert np.array_equal(counts.cpu().numpy(), np.bincount(np.where(codes[:m] <= 11, codes[:m], 15),
                                                                minlength=16))
        want = O.oracle_models(s, rec[:m], args, codes[:m], ctx[:m], kill_ns=1000, save_bytes_per_us=1500)
        assert got == want


@pytest.mark.gpu
def test_gpu_validate_models_c2_fused():
    """C2 and C2 x 24 (the fused kernel's steady state, >= 2 tiles per CTA):
    one launch; verdicts = the oracle's (tiled), models = the oracle's on the
    base trace times 24 (copies are the same instances relocated);
    and the base trace on 64-record tiles (~2 tiles per CTA of 148)."""
    import paper_2410_23661_b200 as pk
    from tracegen import workloads
    s, rec, args, meta = workloads.make_c2()
    codes = np.array(O.oracle_batch_mp(s, rec, args), np.uint8)
    ctx = np.random.default_rng(5).integers(4_000, 98_001, len(rec)).astype(np.uint64)
    want = O.oracle_models(s, rec, args, codes, ctx)
    p = pk.Picker(0)
    p.load(s)
    (flags, _, _), got = p.validate_models(rec, args, ctx)
    assert p.last_launch_count() == 1
    assert np.array_equal(flags.cpu().numpy(), codes)
    assert got == want
    R = 24  # 437 K records: >= 2 tiles of 640 per CTA of the models module
    rec_t, args_t = workloads.replicate(rec, args, meta["ptr_mask"], R)
    (flags, _, _), got = p.validate_models(rec_t, args_t, np.tile(ctx, R))
    assert np.array_equal(flags.cpu().numpy(), np.tile(codes, R))
    want_t = {k: (v * R if isinstance(v, int) else [x * R for x in v]) for k, v in want.items()}
    assert got == want_t
    p.close()
    p = pk.Picker(0, tile=64, threads=64, ctas=1, args_per_rec=4, arg_bufs=1)
    p.load(s)
    (flags, _, _), got = p.validate_models(rec, args, ctx)
    assert p.last_launch_count() == 1
    assert np.array_equal(flags.cpu().numpy(), codes)
    assert got == want


@pytest.mark.gpu
def test_gpu_models_given_codes_c2():
    """picker_consumer_models through the models module's kernel (1 launch):
    the models take the CALLER's verdicts, not the kernel's own -- C2 with the
    oracle's codes rotated by 7 records (every record paired with another
    record's verdict) against oracle_models on the same rotated codes."""
    import paper_2410_23661_b200 as pk
    from tracegen import workloads
    s, rec, args, _ = workloads.make_c2()
    codes = np.roll(np.array(O.oracle_batch_mp(s, rec, args), np.uint8), 7)
    ctx = np.random.default_rng(11).integers(0, 150_000, len(rec)).astype(np.uint64)
    p = pk.Picker(0)
    p.load(s)
    got = p.consumer_models(rec, args, codes, ctx, kill_ns=900, save_bytes_per_us=2500)
    assert p.last_launch_count() == 1
    assert got == O.oracle_models(s, rec, args, codes, ctx, kill_ns=900, save_bytes_per_us=2500)


@pytest.mark.gpu
def test_gpu_validate_models_c2heavy():
    """C2-heavy: fused kernels with up to 29 reads (more than the 12 a
    specialised shape sums itself: those records take the table path inside
    the fused kernel) and the 128-key module."""
    import paper_2410_23661_b200 as pk
    from tracegen import workloads
    s, rec, args, meta = workloads.make_c2(heavy=True)
    codes = np.array(O.oracle_batch_mp(s, rec, args), np.uint8)
    ctx = np.random.default_rng(9).integers(0, 300_000, len(rec)).astype(np.uint64)
    want = O.oracle_models(s, rec, args, codes, ctx, kill_ns=700, save_bytes_per_us=3000)
    p = pk.Picker(0)
    p.load(s)
    (flags, _, _), got = p.validate_models(rec, args, ctx, kill_ns=700, save_bytes_per_us=3000)
    assert p.last_launch_count() == 1
    assert np.array_equal(flags.cpu().numpy(), codes)
    assert got == want


@pytest.mark.gpu
def test_gpu_models_errors():
    """Call errors are statuses, not crashes: save bandwidth 0 -> EINVAL."""
    import paper_2410_23661_b200 as pk
    s = golden.golden_summary()
    b = RecordBuilder()
    b.add(0, [4096, 8192, 12288], (4, 1, 1), (128, 1, 1))
    rec, args = b.build()
    p = pk.Picker(0)
    p.load(s)
    flags, _, _ = p.validate(rec, args)
    with pytest.raises(pk.PickerError) as e:
        p.consumer_models(rec, args, flags, None, save_bytes_per_us=0)
    assert e.value.status == -1
    m = p.consumer_models(rec, args, flags, None)
    assert m["n"] == 1 and m["preempt_ns_without"] == 0 and m["ckpt_bytes_all"] == 2 * 4 * 4 * 128
