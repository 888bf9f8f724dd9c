"""GPU parity of the wide path ("instances with many pointer
arguments use a segmented sort plus a sweep-line interval-intersection
kernel"): kernels with more than 4096 read x write pairs are auto-routed to
K2, where one warp evaluates one record; <= 64 descriptors sort in registers,
<= 1024 in the warp's scratch, beyond that lanes test all pairs.  Codes,
bits and counts against the oracle (the plain pairwise definition)."""
import numpy as np
import pytest
import torch

import oracle.picker_oracle as O
from tracegen import workloads
from tracegen.comb import comb_summary
from tracegen.records import RecordBuilder

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    import paper_2410_23661_b200 as pk
    return pk


def _check(flags, bits, counts, want):
    got = flags.cpu().numpy()
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first at {bad[:8]}: gpu {got[bad[:8]]} oracle {want[bad[:8]]}"
    n = len(want)
    idem = (want <= 1).astype(np.uint8)
    words = np.packbits(np.pad(idem, (0, (-n) % 32)).reshape(-1, 32)[:, ::-1], axis=1).view(">u4")
    assert np.array_equal(bits.cpu().numpy().view(np.uint32), words.reshape(-1).astype(np.uint32))
    assert np.array_equal(counts.cpu().numpy(), np.bincount(np.where(want <= 11, want, 15), minlength=16))


def _run(pk, s, rec, args, **opt):
    p = pk.Picker(0, **opt)
    p.load(s)
    out = p.validate(rec, args)
    paths = p.kernel_paths()
    torch.cuda.synchronize()
    p.close()
    return out, paths


@pytest.fixture(scope="module")
def wide():
    s, rec, args, meta = workloads.make_wide(n=3000)
    return s, rec, args, np.array(O.oracle_batch_mp(s, rec, args), np.uint8)


# wide-only summaries take the K2 persistent kernel (k_wide.cu) by default;
# wide_kernel=0 routes them through the module's schedules / the table path
WIDE_PATHS = [dict(jit=1), dict(jit=1, wide_kernel=0), dict(jit=1, wide_kernel=0, sorted=0),
              dict(jit=1, wide_kernel=0, sorted=0, tile=64, threads=32, ctas=1, args_per_rec=8),
              dict(jit=0, bucket=1), dict(jit=0, wide_kernel=0, bucket=1), dict(jit=0, wide_kernel=0, bucket=0),
              dict(jit=0, force_path=3)]


@pytest.mark.parametrize("opt", WIDE_PATHS, ids=str)
def test_wide_family(pk, wide, opt):
    """Multi-tensor kernels with 150-300 symbolic addresses, every one beyond
    4096 pairs (the specialised module routes all of them to K2)."""
    s, rec, args, want = wide
    (flags, bits, counts), paths = _run(pk, s, rec, args, **opt)
    _check(flags, bits, counts, want)
    assert (want == 10).sum() > 0 and (want == 0).sum() > 0
    if opt.get("jit") and "force_path" not in opt:
        assert set(paths.values()) == {"wide"}, paths


@pytest.mark.parametrize("opt", [dict(), dict(wide_kernel=0)], ids=str)
def test_wide_small_batches(pk, wide, opt):
    """Small batches: the K2 kernel with a partial last chunk, and the
    small-batch kernel (n <= 1024), which runs K2 records warp-cooperatively
    with its own scratch slices."""
    s, rec, args, want = wide
    for n in (1, 31, 33, 1024):
        (flags, bits, counts), _ = _run(pk, s, rec[:n], args, **opt)
        _check(flags, bits, counts, want[:n])


@pytest.fixture(scope="module")
def wide_shuffled():
    """The wide family with every record's pointer arguments permuted among
    themselves: extents out of address order (the K2 kernel's chunk sort runs,
    not only its sortedness test) and many more overlaps."""
    s, rec, args, meta = workloads.make_wide(n=2000, seed=5)
    rng = np.random.default_rng(11)
    args = args.copy()
    mask = meta["ptr_mask"]
    for r in rec:
        o, k = int(r["arg_off"]), int(r["nargs"])
        idx = o + np.nonzero(mask[o:o + k])[0]
        if rng.random() < 0.7:
            args[idx] = args[rng.permutation(idx)]
    want = np.array(O.oracle_batch_mp(s, rec, args), np.uint8)
    return s, rec, args, want


@pytest.mark.parametrize("opt", [dict(), dict(wide_kernel=0), dict(jit=0, force_path=3)], ids=str)
def test_wide_shuffled(pk, wide_shuffled, opt):
    s, rec, args, want = wide_shuffled
    assert (want == 0).sum() > 50 and (want == 10).sum() > 50
    (flags, bits, counts), _ = _run(pk, s, rec, args, **opt)
    _check(flags, bits, counts, want)


def test_wide_kernel_steady_state(pk, wide):
    """The wide family x 40 (120,000 records: >= 1.5 chunks of 32 records per
    warp of the K2 kernel's 148 x 16 warps, so warps carry the argument /
    header pipeline across chunks); expected codes = the base trace's oracle
    codes tiled (pointer relocation)."""
    s, rec, args, want = wide
    _, _, _, meta = workloads.make_wide(n=3000)
    R, A = workloads.replicate(rec, args, meta["ptr_mask"], 40)
    (flags, bits, counts), _ = _run(pk, s, R, A)
    _check(flags, bits, counts, np.tile(want, 40))


def _comb_records(seed):
    rng = np.random.default_rng(seed)
    A = 1 << 40
    b = RecordBuilder()
    for kid, nr, nw, nrand in [(0, 40, 40, 300), (1, 600, 500, 300), (2, 20, 20, 300), (3, 1500, 1500, 6)]:
        for B, n in [(A + 64 * nr, 16), (A + 64 * (nr - 1), 1), (A + 32, 8), (A + 32, 9), (A - 64 * nw, 16),
                     (A, 0)]:
            b.add(kid, [A, B, n], grid=(1,), block=(32,))
        for _ in range(nrand):  # random offsets around the teeth
            d = int(rng.integers(-64 * nr - 64, 64 * nr + 64))
            b.add(kid, [A, A + d, int(rng.integers(0, 17))], grid=(1,), block=(32,))
    return b.build()


@pytest.mark.parametrize("opt", [dict(jit=1), dict(jit=1, wide_pairs=4), dict(jit=0, force_path=3),
                                 dict(jit=0, force_path=3, wide_kernel=0), dict(jit=0, bucket=1)], ids=str)
def test_comb_edges(pk, opt):
    """Touching / overlapping / interleaved teeth: register sort (40
    descriptors, forced wide), the smaller side sorted in the scratch (80,
    1,100), lanes over pairs (3,000)."""
    s = comb_summary()
    rec, args = _comb_records(7)
    want = np.array(O.oracle_batch(s, rec, args), np.uint8)
    for q in range(4):
        assert want[q * 306 if q < 3 else 918:][:6].tolist() == [0, 10, 0, 10, 0, 0]
    (flags, bits, counts), paths = _run(pk, s, rec, args, **opt)
    _check(flags, bits, counts, want)
