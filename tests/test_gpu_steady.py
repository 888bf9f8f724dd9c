"""GPU parity in the persistent kernels' steady state: every CTA runs >= 4
tiles, so the paths that only a second tile reaches (emit of tile t-1 after
tile t's evaluation, argument restaging after the evaluation barrier, the
next tile's key pass, the parity reuse of the per-tile code / count buffers,
mbarrier phases >= 2) are compared against the oracle.

Expected codes come from the oracle only:
* directly, record by record (``oracle_batch_mp``), for traces the oracle
  finishes in seconds;
* for tiled traces, as the base trace's oracle codes tiled: copy r of a
  record is the same instance at another position (the code is
  per instance), or relocated by r * delta on its pointer arguments
  (G9, translation invariance, pinned on the CPU in test_oracle_pins.py).

Also the host-buffer call over more than one 2^22-record chunk with a ragged
last chunk (the histogram of every chunk must be summed)."""
import numpy as np
import pytest
import torch

import oracle.picker_oracle as O
from tracegen import workloads
from tracegen.synth import random_records, random_summary

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    import paper_2410_23661_b200 as pk
    return pk


@pytest.fixture(scope="module")
def c2():
    s, rec, args, meta = workloads.make_c2()
    want = np.array(O.oracle_batch_mp(s, rec, args), np.uint8)
    return s, rec, args, meta, want


def _expect_bits_counts(want):
    n = len(want)
    idem = (want <= 1).astype(np.uint8)
    words = np.packbits(np.pad(idem, (0, (-n) % 32)).reshape(-1, 32)[:, ::-1], axis=1).view(">u4")
    cnt = np.bincount(np.where(want <= 11, want, 15), minlength=16).astype(np.int64)
    return words.reshape(-1).astype(np.uint32), cnt


def _check(flags, bits, counts, want):
    got = flags.cpu().numpy() if torch.is_tensor(flags) else flags
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first at {bad[:8]}: gpu {got[bad[:8]]} oracle {want[bad[:8]]}"
    w, c = _expect_bits_counts(want)
    if bits is not None:
        assert np.array_equal(bits.cpu().numpy().view(np.uint32), w)
    if counts is not None:
        assert np.array_equal(counts.cpu().numpy(), c)


def _run(pk, s, rec, args, **opt):
    p = pk.Picker(0, **opt)
    p.load(s)
    out = p.validate(rec, args)
    torch.cuda.synchronize()
    p.close()
    return out


C2_PATHS = [
    dict(jit=1),                                  # auto: 896-record tiles, 2 CTAs/SM
    dict(jit=1, tile=448, threads=224, ctas=4, args_per_rec=5, arg_bufs=1),
    dict(jit=1, tile=448, threads=224, ctas=3, args_per_rec=5, arg_bufs=2),
    dict(jit=0, bucket=1),                        # table path, grouped by kernel (549 keys)
    dict(jit=0, bucket=0),                        # table path, thread per record
]


@pytest.mark.parametrize("opt", C2_PATHS, ids=str)
def test_c2_tiled_steady_state(pk, c2, opt):
    """C2 x 64 = 1,165,888 records: >= 4 tiles per CTA at every geometry."""
    s, rec, args, meta, want = c2
    R = 64
    rec_t, args_t = workloads.replicate(rec, args, meta["ptr_mask"], R)
    flags, bits, counts = _run(pk, s, rec_t, args_t, **opt)
    _check(flags, bits, counts, np.tile(want, R))


GEOMS = [
    dict(jit=1, tile=64, threads=32, ctas=1, args_per_rec=5, arg_bufs=1),
    dict(jit=1, tile=64, threads=32, ctas=1, args_per_rec=5, arg_bufs=2),
    dict(jit=1, tile=64, threads=64, ctas=1, args_per_rec=2, arg_bufs=1),  # spans overflow the buffer
    dict(jit=1, tile=128, threads=64, ctas=1, args_per_rec=3, arg_bufs=2),
]


@pytest.mark.parametrize("opt", GEOMS, ids=str)
def test_random_direct_steady_state(pk, opt):
    """60,001 random records (every IR feature) at 64/128-record tiles on 148
    CTAs: 3-6 tiles per CTA, each code checked directly against the oracle."""
    s = random_summary(41, n_kernels=30)
    rec, args = random_records(42, s, 60001, max_threads=256, max_grid=32)
    want = np.array(O.oracle_batch_mp(s, rec, args), np.uint8)
    flags, bits, counts = _run(pk, s, rec, args, **opt)
    _check(flags, bits, counts, want)


@pytest.mark.parametrize("opt", [dict(jit=1), dict(jit=0, bucket=1), dict(jit=0, bucket=0),
                                 dict(jit=1, tile=64, threads=32, ctas=1, args_per_rec=2, arg_bufs=2)],
                         ids=str)
def test_random_tiled_steady_state(pk, opt):
    """A 7,001-record random trace tiled 100x (copies at other positions, same
    arguments): 700,100 records, >= 4 tiles per CTA on the table path's
    512-record tiles too."""
    s = random_summary(43, n_kernels=30)
    rec, args = random_records(44, s, 7001, max_threads=256, max_grid=32)
    want = np.array(O.oracle_batch_mp(s, rec, args), np.uint8)
    R = 100
    rec_t, args_t = workloads.replicate(rec, args, np.zeros(len(args), bool), R, delta=0)
    flags, bits, counts = _run(pk, s, rec_t, args_t, **opt)
    _check(flags, bits, counts, np.tile(want, R))


def test_c4_tiled_steady_state(pk):
    """C4 x 256 = 1,048,576 records on the shape-sorted schedule (the default
    for many-argument summaries: ~32,800 claimed groups over 148 CTAs) and on
    the tiled kernel (2560-record tiles, 148 CTAs: ~2.8 tiles per CTA; plus
    64-record tiles, >100 per CTA)."""
    s, rec, args, meta = workloads.make_c4(n=1 << 12)
    want = np.array(O.oracle_batch_mp(s, rec, args), np.uint8)
    for R, opt in [(256, dict(jit=1)), (256, dict(jit=1, sort_ws=1)), (256, dict(jit=1, sorted=0)),
                   (8, dict(jit=1, sorted=0, tile=64, threads=32, ctas=1, args_per_rec=20))]:
        rec_t, args_t = workloads.replicate(rec, args, meta["ptr_mask"], R)
        flags, bits, counts = _run(pk, s, rec_t, args_t, **opt)
        _check(flags, bits, counts, np.tile(want, R))


def test_host_call_many_chunks(pk, c2):
    """picker_validate_batch_host over 2^22 + 100 records: two chunks; before
    the fix the last (<= 1024-record) chunk took the small-batch kernel, which
    wrote the counts instead of adding to them."""
    s, rec, args, meta, want = c2
    n = (1 << 22) + 100
    R = -(-n // len(rec))
    rec_t, args_t = workloads.replicate(rec, args, meta["ptr_mask"], R)
    rec_t = rec_t[:n]
    args_t = args_t[: int(rec_t[-1]["arg_off"]) + int(rec_t[-1]["nargs"])]
    p = pk.Picker(0)
    p.load(s)
    rec_h = torch.from_numpy(rec_t.view(np.uint8).reshape(-1, 32)).pin_memory()
    args_h = torch.from_numpy(args_t).pin_memory()
    flags, bits, counts = p.validate_host(rec_h, args_h)
    p.close()
    _check(flags.numpy(), bits, counts, np.tile(want, R)[:n])


@pytest.mark.parametrize("opt", [dict(jit=1), dict(jit=0, bucket=1)], ids=str)
def test_contradictory_preconditions(pk, opt):
    """a kernel whose precondition box is empty loads and
    every one of its records is code 7, next to a kernel
    on the specialised path."""
    from tracegen import golden
    from tracegen.records import RecordBuilder
    k = golden.relu(0)
    k["pre"] = [p for p in k["pre"] if p["op"] != "N"] + [{"op": "N", "lo": 5, "hi": 3}]
    s = {"version": 1, "kernels": [k, golden.vector_add(1)]}
    b = RecordBuilder()
    for i in range(3000):
        if i % 3:
            b.add(0, (0x10000, 0x20000, 16 + i % 20), grid=(4,), block=(32,))
        else:
            b.add(1, (0x1000, 0x2000, 0x3000 if i % 2 else 0x1000), grid=(4,), block=(128,))
    rec, args = b.build()
    want = np.array(O.oracle_batch(s, rec, args), np.uint8)
    assert set(want[1::3]) == {7}
    flags, bits, counts = _run(pk, s, rec, args, **opt)
    _check(flags, bits, counts, want)


def test_device_replication(pk, c2):
    """K6 (picker_replicate) writes exactly the host generator's relocated
    copies (tracegen.workloads.replicate), and their verdicts are the base
    trace's tiled."""
    s, rec, args, meta, want = c2
    p = pk.Picker(0)
    p.load(s)
    R, first = 7, 3
    rd, ad = p.replicate(rec, args, meta["ptr_mask"], R, first_copy=first, delta=1 << 37)
    hr, ha = workloads.replicate(rec, args, meta["ptr_mask"], R + first)
    hr, ha = hr[first * len(rec):], ha[first * len(args):]  # host copies first .. first + R - 1
    got = rd.cpu().numpy().reshape(-1).view(hr.dtype)
    for f in hr.dtype.names:  # device copy c: arg_off + c * len(args); host copy first + c
        want_f = hr[f] - first * len(args) if f == "arg_off" else hr[f]
        assert np.array_equal(got[f], want_f), f
    assert np.array_equal(ad.cpu().numpy(), ha)
    flags, bits, counts = p.validate(rd, ad)
    _check(flags, bits, counts, np.tile(want, R))
    p.close()


def test_c2heavy_128_keys(pk):
    """C2-heavy has 66 shapes: the pipelined kernel with 128 grouping keys (4
    per lane in the scan), every record against the oracle, many tiles per CTA:
    the auto geometry for > 64 keys (1792-record tiles, one CTA of 896 threads
    per SM; x80 = 5.5 tiles per CTA) and the few-key geometry (2 x 448 on 896)."""
    s, rec, args, meta = workloads.make_c2(heavy=True)
    want = np.array(O.oracle_batch_mp(s, rec, args), np.uint8)
    for R, opt in [(1, dict(jit=1)), (80, dict(jit=1)),
                   (40, dict(jit=1, tile=896, threads=448, ctas=2, args_per_rec=5, arg_bufs=1)),
                   (4, dict(jit=1, tile=64, threads=32, ctas=1, args_per_rec=8))]:
        rec_t, args_t = workloads.replicate(rec, args, meta["ptr_mask"], R)
        flags, bits, counts = _run(pk, s, rec_t, args_t, **opt)
        _check(flags, bits, counts, np.tile(want, R))
