"""GPU parity: verdict codes from the CUDA path, through the C ABI, are
byte-identical to the CPU oracle on the same seeded inputs (integer work:
bit-exact).  Also checks the packed idempotent bits and the histogram."""
import json
import os

import numpy as np
import pytest
import torch

import oracle.picker_oracle as O
from tracegen import golden
from tracegen.records import RecordBuilder, concat
from tracegen.synth import random_records, random_summary

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(__file__)


@pytest.fixture(scope="module")
def pk():
    import paper_2410_23661_b200 as pk
    return pk


def _make(pk, summary, **opt):
    p = pk.Picker(0, **opt)
    p.load(summary)
    return p


def _oracle_codes(summary, rec, args, fn=O.oracle_interval, **kw):
    return np.array(O.oracle_batch_mp(summary, rec, args, fn, **kw), dtype=np.uint8)


def _check_outputs(flags, bits, counts, want):
    got = flags.cpu().numpy()
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first at {bad[:8]}: gpu {got[bad[:8]]} oracle {want[bad[:8]]}"
    n = len(want)
    idem = (want <= 1).astype(np.uint8)
    exp_bits = np.packbits(np.pad(idem, (0, (-n) % 32)).reshape(-1, 32)[:, ::-1], axis=1)
    exp_words = exp_bits.view(">u4").reshape(-1).astype(np.uint32)
    if bits is not None:
        assert np.array_equal(bits.cpu().numpy().view(np.uint32), exp_words)
    if counts is not None:
        exp_c = np.zeros(16, np.int64)
        for c in want:
            exp_c[c if c <= 11 else 15] += 1
        assert np.array_equal(counts.cpu().numpy(), exp_c)


PATH_OPTS = [dict(jit=0, bucket=0), dict(jit=0, bucket=1), dict(jit=1),
             dict(jit=0, force_path=3), dict(jit=1, wide_pairs=4)]


@pytest.mark.parametrize("opt", PATH_OPTS, ids=str)
def test_paper_examples(pk, opt):
    s = golden.golden_summary()
    cases = json.load(open(os.path.join(HERE, "golden", "paper_examples.json")))["cases"]
    b = RecordBuilder()
    for c in cases:
        b.add(c["kernel_id"], c["args"], c["grid"], c["block"])
    rec, args = b.build()
    p = _make(pk, s, **opt)
    flags, bits, counts = p.validate(rec, args)
    want = np.array([c["interval"] for c in cases], np.uint8)
    _check_outputs(flags, bits, counts, want)


@pytest.mark.parametrize("opt", PATH_OPTS, ids=str)
def test_c1_vector_add(pk, opt):
    s = {"version": 1, "kernels": [golden.vector_add()]}
    rec, args = golden.c1_records()
    p = _make(pk, s, **opt)
    flags, bits, counts = p.validate(rec, args)
    _check_outputs(flags, bits, counts, np.array([0, 10, 10, 0, 0, 10, 10, 7], np.uint8))


@pytest.mark.parametrize("opt", PATH_OPTS, ids=str)
@pytest.mark.parametrize("seed", [101, 102, 103, 104])
def test_random_small(pk, opt, seed):
    """Randomized summaries (all IR features) x records spanning many CTA tiles
    with a ragged tail; byte-equal codes vs the oracle."""
    s = random_summary(seed, n_kernels=40)
    rec, args = random_records(seed + 7, s, 5000 + seed % 97, max_threads=256, max_grid=64)
    want = _oracle_codes(s, rec, args)
    p = _make(pk, s, **opt)
    flags, bits, counts = p.validate(rec, args)
    _check_outputs(flags, bits, counts, want)


@pytest.mark.parametrize("opt", PATH_OPTS, ids=str)
def test_random_large_ranges(pk, opt):
    """Large preconditions (64-bit extents, big grids) -- the oracle's
    endpoint path and the loader's wrap-freedom proof at scale."""
    s = random_summary(7, n_kernels=40, small=False)
    rec, args = random_records(8, s, 4000, max_threads=1024, max_grid=65535)
    want = _oracle_codes(s, rec, args)
    p = _make(pk, s, **opt)
    flags, bits, counts = p.validate(rec, args)
    _check_outputs(flags, bits, counts, want)


def test_empty_and_tiny_batches(pk):
    s = golden.golden_summary()
    p = _make(pk, s)
    rec, args = golden.c1_records()
    for n in (0, 1, 31, 32, 33):
        r = np.resize(rec, n) if n else rec[:0]
        flags, bits, counts = p.validate(r, args)
        want = _oracle_codes(s, r, args)
        _check_outputs(flags, bits, counts, want)


def test_host_path_matches(pk):
    s = random_summary(5, n_kernels=30)
    rec, args = random_records(6, s, 3000, max_threads=128, max_grid=16)
    want = _oracle_codes(s, rec, args)
    p = _make(pk, s)
    rt = torch.from_numpy(rec.view(np.uint8).reshape(-1, 32)).pin_memory()
    at = torch.from_numpy(args).pin_memory()
    flags, bits, counts = p.validate_host(rt, at)
    _check_outputs(flags, bits, counts, want)
    flags, bits, counts = p.validate_host(rt, at, packed=False)
    _check_outputs(flags, bits, counts, want)


def test_unpacked_args(pk):
    """arg_off in any order (args_packed = 0)."""
    s = random_summary(9, n_kernels=20)
    rec, args = random_records(10, s, 2000, max_threads=64, max_grid=8)
    perm = np.random.default_rng(0).permutation(len(rec))
    rec2 = rec[perm]
    want = _oracle_codes(s, rec2, args)
    p = _make(pk, s)
    flags, bits, counts = p.validate(rec2, args, packed=False)
    _check_outputs(flags, bits, counts, want)


# ---- K3 exact verifier (picker_exact_check) vs oracle_exact ---------------------

def test_exact_paper_examples(pk):
    s = golden.golden_summary()
    cases = json.load(open(os.path.join(HERE, "golden", "paper_examples.json")))["cases"]
    b = RecordBuilder()
    for c in cases:
        b.add(c["kernel_id"], c["args"], c["grid"], c["block"])
    rec, args = b.build()
    p = _make(pk, s)
    out, counts = p.exact_check(rec, args)
    want = np.array([c["exact"] for c in cases], np.uint8)
    assert np.array_equal(out.cpu().numpy(), want), (out.cpu().numpy(), want)
    exp_c = np.zeros(16, np.int64)
    for c in want:
        exp_c[c if c <= 11 else 15] += 1
    assert np.array_equal(counts.cpu().numpy(), exp_c)


@pytest.mark.parametrize("seed", [201, 202, 203])
def test_exact_random(pk, seed):
    """Byte-set intersection on the GPU == the oracle's Python sets, including
    the point cap (code 11) and range-overestimation records (interval 10,
    exact 0)."""
    cap = 1 << 12
    s = random_summary(seed, n_kernels=30)
    rec, args = random_records(seed + 5, s, 1500, max_threads=32, max_grid=4)
    want = _oracle_codes(s, rec, args, O.oracle_exact, cap=cap)
    inter = _oracle_codes(s, rec, args)
    p = _make(pk, s)
    out, _ = p.exact_check(rec, args, max_points=cap)
    got = out.cpu().numpy()
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, (bad[:8], got[bad[:8]], want[bad[:8]])
    # range overestimation exists in these traces and is measured exactly
    assert ((inter == 10) & (got == 0)).sum() > 0
    # no false positives: interval idempotent => exact idempotent
    assert not ((inter == 0) & (got == 10)).any()


def test_exact_cap_boundary_and_far_windows(pk):
    """Code 11 at the point-cap boundary (1,536 points: cap 1,535 -> 11, cap
    1,536 -> verdict), and accesses 2^36 bytes apart whose shared window spans
    ~3 x 2^36 bytes (the byte-set tables hold only touched 64-byte blocks)."""
    from test_oracle_pins import far_stride_summary
    s = golden.golden_summary()
    b = RecordBuilder()
    b.add(0, [0x1000, 0x2000, 0x3000], (4,), (128,))
    b.add(0, [0x1000, 0x2000, 0x1000], (4,), (128,))
    rec, args = b.build()
    p = _make(pk, s)
    for cap, want in [(1535, [11, 11]), (1536, [0, 10])]:
        out, _ = p.exact_check(rec, args, max_points=cap)
        assert out.cpu().numpy().tolist() == want
        assert _oracle_codes(s, rec, args, O.oracle_exact, cap=cap).tolist() == want
    s = far_stride_summary()
    b = RecordBuilder()
    for off in range(0, 9):
        for S in (1 << 36, 1 << 40, 64, 8, 4):
            b.add(0, [1 << 44, S, off], (1,), (4,))
            b.add(0, [1 << 44, S, off], (1,), (1024,))
    rec, args = b.build()
    want = _oracle_codes(s, rec, args, O.oracle_exact)
    p = _make(pk, s)
    out, _ = p.exact_check(rec, args)
    assert np.array_equal(out.cpu().numpy(), want)
    assert (want == 0).sum() > 0 and (want == 10).sum() > 0


def test_exact_big_tables(pk):
    """Records whose written blocks exceed a CTA slice of the small pass
    (65,536 threads writing every 64th byte: > 2^16 table entries) take the
    big pass; with and without a shared byte."""
    t = {"gidx.x": {"lo": [], "hi": []}}
    k = golden.kernel(
        0, "spread", [("A", "ptr"), ("S", "i64"), ("off", "i64")],
        [golden.desc("R", 4, "A", [golden.term(1, ["S"], "gidx.x")], t),
         golden.desc("W", 4, "A", [golden.term(1, ["S"], "gidx.x"), golden.term(1, ["off"])], t)],
        pre=golden.ptr_pre("A") + [{"op": "S", "lo": 0, "hi": 1 << 20}, {"op": "off", "lo": 0, "hi": 1 << 30}])
    s = {"version": 1, "kernels": [k]}
    b = RecordBuilder()
    for S, off in [(64, 4), (64, 3), (128, 64), (128, 128), (64, 64 * 65535 + 4), (64, 64 * 65535)]:
        b.add(0, [1 << 40, S, off], (64,), (1024,))
    rec, args = b.build()
    want = _oracle_codes(s, rec, args, O.oracle_exact)
    assert want.tolist() == [0, 10, 0, 10, 0, 10]
    p = _make(pk, s)
    out, _ = p.exact_check(rec, args)
    assert np.array_equal(out.cpu().numpy(), want)


# ---- C4: cuDNN-like kernels with 16-48 pointer arguments ------------------------

@pytest.mark.parametrize("opt", [dict(jit=1), dict(jit=1, sorted=0), dict(jit=1, force_path=3),
                                 dict(jit=1, force_path=3, sorted=0), dict(jit=0, force_path=3),
                                 dict(jit=0, bucket=0)], ids=str)
def test_c4_many_pointers(pk, opt):
    """Specialised pairwise, the K2 sort+sweep path and the table path agree
    with the oracle on cuDNN-like records (sweep == pairwise)."""
    from tracegen.workloads import make_c4
    s, rec, args, _ = make_c4(n=3000, n_kernels=12)
    want = _oracle_codes(s, rec, args)
    p = _make(pk, s, **opt)
    flags, bits, counts = p.validate(rec, args)
    _check_outputs(flags, bits, counts, want)
    assert (want == 10).sum() > 0 and (want == 0).sum() > 0


@pytest.mark.parametrize("opt", [dict(jit=0), dict(jit=1)], ids=str)
def test_c2_trace_every_record(pk, opt):
    """The C2 trace (547 kernels): with the specialised module off the
    table-driven path groups by kernel (549 keys: k_validate_bucket); on, by
    shape (35 keys: k_validate_pipe).  Every record against the oracle."""
    from tracegen import workloads
    s, rec, args, _ = workloads.make_c2()
    p = _make(pk, s, **opt)
    flags, bits, counts = p.validate(rec, args)
    _check_outputs(flags, bits, counts, _oracle_codes(s, rec, args))
