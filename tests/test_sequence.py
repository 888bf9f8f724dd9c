"""Multi-kernel idempotency: oracle pins
(CPU) and GPU parity of picker_validate_sequence."""
import numpy as np
import pytest

import oracle.picker_oracle as O
from tracegen import golden
from tracegen.records import RecordBuilder
from tracegen.synth import random_records, random_summary

G = O.index_summary(golden.golden_summary())


def _recs(rows):
    b = RecordBuilder()
    for kid, args, grid, block in rows:
        b.add(kid, args, grid=grid, block=block)
    rec, args = b.build()
    return [O.decode_record(r, args) for r in rec]


VA = dict(grid=(4, 1, 1), block=(128, 1, 1))  # vectorAdd: A = B + C, 0x800-byte buffers


def _va(a, b, c):
    return (0, [a, b, c], VA["grid"], VA["block"])


def test_clobber_of_an_earlier_read():
    """k1: A1 = B1 + C1; k2: B1 = A1 + C1 -- k2 overwrites B1, an input of k1:
    a clobber anti-dependency across the list."""
    r = _recs([_va(0x10000, 0x20000, 0x30000), _va(0x20000, 0x10000, 0x30000)])
    assert O.oracle_sequence(G, r, O.SEQ_SEQUENTIAL) == O.NI_OVERLAP
    assert O.oracle_sequence(G, r, O.SEQ_CONCURRENT) == O.NI_OVERLAP


def test_read_after_write_is_not_a_clobber():
    """k1: A = B + C; k2: D = A + C -- k2 reads what k1 wrote (RAW), no input of
    the list is overwritten: idempotent as a sequence, but not as a concurrent set
    (concurrent = any read/write overlap)."""
    r = _recs([_va(0x10000, 0x20000, 0x30000), _va(0x40000, 0x10000, 0x30000)])
    assert O.oracle_sequence(G, r, O.SEQ_SEQUENTIAL) == O.IDEM_CHECKED
    assert O.oracle_sequence(G, r, O.SEQ_CONCURRENT) == O.NI_OVERLAP


def test_disjoint_list_is_idempotent():
    r = _recs([_va(0x10000 * (3 * i + 1), 0x10000 * (3 * i + 2), 0x10000 * (3 * i + 3)) for i in range(5)])
    for m in (O.SEQ_SEQUENTIAL, O.SEQ_CONCURRENT):
        assert O.oracle_sequence(G, r, m) == O.IDEM_CHECKED


def test_write_only_kernel_clobbers_earlier_input():
    """vectorSet (kernel-level idempotent alone) still overwrites a byte read by an
    earlier instance of the list."""
    r = _recs([_va(0x10000, 0x20000, 0x30000), (1, [0x20000], VA["grid"], VA["block"])])
    assert O.oracle_sequence(G, r) == O.NI_OVERLAP
    r = _recs([(1, [0x20000], VA["grid"], VA["block"]), _va(0x10000, 0x20000, 0x30000)])
    assert O.oracle_sequence(G, r) == O.IDEM_CHECKED  # the set happens first: RAW


def test_first_decisive_instance_decides():
    r = _recs([_va(0x10000, 0x20000, 0x30000), (2, [0x50000], VA["grid"], VA["block"]),
               _va(1 << 56, 0x20000, 0x30000)])
    assert O.oracle_sequence(G, r) == 2  # vectorInc (SO) precedes the precondition failure


def test_window_of_one_matches_single_instance():
    s = random_summary(5, n_kernels=20)
    rec, args = random_records(6, s, 300, max_threads=16, max_grid=2)
    w1 = O.oracle_windows(s, rec, args, 1)
    iv = O.oracle_batch(s, rec, args)
    for a, b in zip(w1, iv):
        assert a == b or (a, b) == (0, 1)  # a write-only kernel is idempotent either way


@pytest.mark.gpu
@pytest.mark.parametrize("window", [1, 3, 8, 32])
@pytest.mark.parametrize("concurrent", [False, True])
def test_gpu_sequence_parity(window, concurrent):
    import paper_2410_23661_b200 as pk
    s = random_summary(31, n_kernels=24)
    rec, args = random_records(32, s, 2000 + window, max_threads=32, max_grid=4)
    want = np.array(O.oracle_windows(s, rec, args, window, O.SEQ_CONCURRENT if concurrent else O.SEQ_SEQUENTIAL),
                    np.uint8)
    p = pk.Picker(0)
    p.load(s)
    got = p.validate_sequence(rec, args, window, concurrent=concurrent).cpu().numpy()
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, (bad[:8], got[bad[:8]], want[bad[:8]])
    assert len(set(want.tolist())) > 2


# Opaque windows (reading Q23 with the opaque rule of PAPER.md l.761-765).
# Kernel 9 (opaque_io): rflag 1 = plain read src+4*tid, 2 = opaque read;
# wflag 1 = opaque write, 2 = plain write out+4*tid.  bdim 32: 128-byte extents.
def _io(out, src, rflag, wflag):
    return (9, [out, src, rflag, wflag], (1, 1, 1), (32, 1, 1))


def test_opaque_write_after_a_read():
    """Instance 0 reads src, instance 1 writes through an opaque address: the
    write may clobber the earlier input (j=1 >= i=0) -> 9 in both modes."""
    r = _recs([_io(0x10000, 0x20000, 1, 0), _io(0x30000, 0x40000, 0, 1)])
    assert O.oracle_sequence(G, r, O.SEQ_SEQUENTIAL) == O.NI_OPAQUE
    assert O.oracle_sequence(G, r, O.SEQ_CONCURRENT) == O.NI_OPAQUE


def test_opaque_write_before_a_read():
    """The opaque write comes first: a later read sees the written value (RAW),
    no input of the list is clobbered -> 0 sequential; concurrent -> 9."""
    r = _recs([_io(0x30000, 0x40000, 0, 1), _io(0x10000, 0x20000, 1, 0)])
    assert O.oracle_sequence(G, r, O.SEQ_SEQUENTIAL) == O.IDEM_CHECKED
    assert O.oracle_sequence(G, r, O.SEQ_CONCURRENT) == O.NI_OPAQUE


def test_opaque_read_before_a_write():
    """Instance 0 reads through an opaque address, instance 1 writes out: the
    write may clobber what was read -> 9 in both modes."""
    r = _recs([_io(0x10000, 0x20000, 2, 0), _io(0x30000, 0x40000, 0, 2)])
    assert O.oracle_sequence(G, r, O.SEQ_SEQUENTIAL) == O.NI_OPAQUE
    assert O.oracle_sequence(G, r, O.SEQ_CONCURRENT) == O.NI_OPAQUE


def test_opaque_read_after_a_write():
    """The plain write comes first, the opaque read after it -> 0 sequential
    (RAW); concurrent -> 9."""
    r = _recs([_io(0x30000, 0x40000, 0, 2), _io(0x10000, 0x20000, 2, 0)])
    assert O.oracle_sequence(G, r, O.SEQ_SEQUENTIAL) == O.IDEM_CHECKED
    assert O.oracle_sequence(G, r, O.SEQ_CONCURRENT) == O.NI_OPAQUE


def test_opaque_inside_one_instance():
    """One instance with an opaque write and a plain read is 9 as a window of
    one, as it is alone (test golden 'opaque write with an active read')."""
    r = _recs([_io(0x10000, 0x20000, 1, 1)])
    for m in (O.SEQ_SEQUENTIAL, O.SEQ_CONCURRENT):
        assert O.oracle_sequence(G, r, m) == O.NI_OPAQUE
    r = _recs([_io(0x10000, 0x20000, 0, 1), _io(0x50000, 0x60000, 0, 1)])  # writes only
    for m in (O.SEQ_SEQUENTIAL, O.SEQ_CONCURRENT):
        assert O.oracle_sequence(G, r, m) == O.IDEM_CHECKED


@pytest.mark.gpu
@pytest.mark.parametrize("concurrent", [False, True])
def test_gpu_sequence_golden_opaque(concurrent):
    """The hand-derived opaque windows above, through picker_validate_sequence."""
    import paper_2410_23661_b200 as pk
    rows = [_io(0x10000, 0x20000, 1, 0), _io(0x30000, 0x40000, 0, 1),
            _io(0x30000, 0x40000, 0, 1), _io(0x10000, 0x20000, 1, 0),
            _io(0x10000, 0x20000, 2, 0), _io(0x30000, 0x40000, 0, 2),
            _io(0x30000, 0x40000, 0, 2), _io(0x10000, 0x20000, 2, 0),
            _io(0x10000, 0x20000, 0, 1), _io(0x50000, 0x60000, 0, 1)]
    want = [9, 9, 9, 9, 0] if concurrent else [9, 0, 9, 0, 0]
    b = RecordBuilder()
    for kid, a, grid, block in rows:
        b.add(kid, a, grid=grid, block=block)
    rec, args = b.build()
    p = pk.Picker(0)
    p.load(golden.golden_summary())
    got = p.validate_sequence(rec, args, 2, concurrent=concurrent).cpu().numpy()
    assert got.tolist() == want


@pytest.mark.gpu
@pytest.mark.parametrize("window", [32, 1024])
@pytest.mark.parametrize("concurrent", [False, True])
@pytest.mark.parametrize("k1", ["lazy", "extents", "tables"])
def test_gpu_sequence_c2(window, concurrent, k1):
    """The C2 trace (547 kernels) cut into windows of 32 / 1024 launches: every
    window's code against oracle_windows (sort + sweep passes vs the plain
    pairwise definition) -- on K1's verdicts and extents (the specialised
    kernels write them, the window kernel reads them: 2 launches) and on the
    tables (1 launch)."""
    import paper_2410_23661_b200 as pk
    from tracegen import workloads
    s, rec, args, _ = workloads.make_c2()
    mode = O.SEQ_CONCURRENT if concurrent else O.SEQ_SEQUENTIAL
    want = np.array(O.oracle_windows(s, rec, args, window, mode), np.uint8)
    opts = {"lazy": dict(seq_lazy=1), "extents": dict(seq_lazy=0), "tables": dict(seq_k1=0)}[k1]
    p = pk.Picker(0, **opts)
    p.load(s)
    got = p.validate_sequence(rec, args, window, concurrent=concurrent).cpu().numpy()
    # windows of 32: decided inside K1's kernel (from its codes, or in the
    # extents module from its extents: 1 launch); of 1024: the extents arena,
    # then the window kernel (2)
    assert p.last_launch_count() == (2 if k1 != "tables" and window > 32 else 1)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, (bad[:8], got[bad[:8]], want[bad[:8]])
    assert len(set(want.tolist())) > 2
    # the C2 records that reach the address check on their own (codes 0, 9,
    # 10): windows decided by the sort + sweep passes, not by a decisive record
    codes = np.array(O.oracle_batch(s, rec, args), np.uint8)
    keep = np.isin(codes, [0, 9, 10])
    sub = rec[keep]
    w2 = 16 if window == 32 else 64
    want = np.array(O.oracle_windows(s, sub, args, w2, mode), np.uint8)
    got = p.validate_sequence(sub, args, w2, concurrent=concurrent).cpu().numpy()
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, (bad[:8], got[bad[:8]], want[bad[:8]])
    assert (want == 0).sum() > 0 and (want == 10).sum() > 0


@pytest.mark.gpu
@pytest.mark.parametrize("concurrent", [False, True])
def test_gpu_sequence_wide(concurrent):
    """Windows of multi-tensor kernels with 150-300 descriptors (no limit on
    descriptors per kernel) and of the comb kernels (touching / interleaved
    teeth across instances)."""
    import paper_2410_23661_b200 as pk
    from tracegen import workloads
    from tracegen.comb import comb_summary
    mode = O.SEQ_CONCURRENT if concurrent else O.SEQ_SEQUENTIAL
    s, rec, args, _ = workloads.make_wide(n=96)
    for window in (2, 5):
        want = np.array(O.oracle_windows(s, rec, args, window, mode), np.uint8)
        p = pk.Picker(0)
        p.load(s)
        got = p.validate_sequence(rec, args, window, concurrent=concurrent).cpu().numpy()
        assert np.array_equal(got, want), (np.nonzero(got != want)[0][:8])
    s = comb_summary()
    rng = np.random.default_rng(5)
    b = RecordBuilder()
    A = 1 << 40
    for i in range(64):
        kid = int(rng.integers(0, 3))
        nr = [40, 600, 20][kid]
        b.add(kid, [A + 64 * int(rng.integers(-nr, nr)), A + 64 * int(rng.integers(-nr, nr)) + int(rng.integers(0, 64)),
                    int(rng.integers(0, 17))], grid=(1,), block=(32,))
    rec, args = b.build()
    for window in (1, 3, 8):
        want = np.array(O.oracle_windows(s, rec, args, window, mode), np.uint8)
        p = pk.Picker(0)
        p.load(s)
        got = p.validate_sequence(rec, args, window, concurrent=concurrent).cpu().numpy()
        assert np.array_equal(got, want), (window, np.nonzero(got != want)[0][:8])


@pytest.mark.gpu
@pytest.mark.parametrize("concurrent", [False, True])
def test_gpu_sequence_k1_tiles(concurrent):
    """The extents module on 64-record tiles (285 tiles over 148 CTAs: the
    restaging / next-tile key pass paths) for the C2 trace: windows of 32
    decided in its kernel (1 launch), and windows of 24 (not dividing the
    tile: its extents arena, then the window kernel), against oracle_windows."""
    import paper_2410_23661_b200 as pk
    from tracegen import workloads
    s, rec, args, _ = workloads.make_c2()
    mode = O.SEQ_CONCURRENT if concurrent else O.SEQ_SEQUENTIAL
    want = np.array(O.oracle_windows(s, rec, args, 32, mode), np.uint8)
    p = pk.Picker(0, tile=64, threads=64, ctas=1, args_per_rec=4, arg_bufs=1)
    p.load(s)
    got = p.validate_sequence(rec, args, 32, concurrent=concurrent).cpu().numpy()
    assert p.last_launch_count() == 1
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, (bad[:8], got[bad[:8]], want[bad[:8]])
    want = np.array(O.oracle_windows(s, rec, args, 24, mode), np.uint8)
    got = p.validate_sequence(rec, args, 24, concurrent=concurrent).cpu().numpy()
    assert p.last_launch_count() == 2
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, (bad[:8], got[bad[:8]], want[bad[:8]])


@pytest.mark.gpu
@pytest.mark.parametrize("concurrent", [False, True])
@pytest.mark.parametrize("lazy", [1, 0, -1], ids=["lazy", "extents", "auto"])
def test_gpu_sequence_fused_steady(concurrent, lazy):
    """Windows decided inside the extents module's pipelined kernel, at its
    steady state (C2 cut to a multiple of 32 records, x 24: ~3 tiles per CTA, so
    windows of tile t run while tile t + 1 is staged and sorted): one launch,
    every window equal to the oracle's windows of the base trace, tiled (the
    copies are the base instances relocated); then windows of 8
    and 16, and a ragged last window.  Lazy: from K1's codes, extents only for
    the windows without a decisive record; extents: K1's extents in shared
    memory; auto: chosen by the first call."""
    import paper_2410_23661_b200 as pk
    from tracegen import workloads
    s, rec, args, meta = workloads.make_c2()
    mode = O.SEQ_CONCURRENT if concurrent else O.SEQ_SEQUENTIAL
    rec = rec[: len(rec) // 32 * 32]
    R = 24
    rec_t, args_t = workloads.replicate(rec, args, meta["ptr_mask"], R)
    p = pk.Picker(0, seq_lazy=lazy)
    p.load(s)
    for window in (32, 16, 8):
        want = np.array(O.oracle_windows(s, rec, args, window, mode), np.uint8)
        got = p.validate_sequence(rec_t, args_t, window, concurrent=concurrent).cpu().numpy()
        assert p.last_launch_count() == 1
        bad = np.nonzero(got != np.tile(want, R))[0]
        assert bad.size == 0, (window, bad[:8], got[bad[:8]])
    m = len(rec) - 13  # ragged: the last window has 19 launches
    want = np.array(O.oracle_windows(s, rec[:m], args, 32, mode), np.uint8)
    got = p.validate_sequence(rec[:m], args, 32, concurrent=concurrent).cpu().numpy()
    assert np.array_equal(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("lazy", [1, -1], ids=["lazy", "auto"])
def test_gpu_sequence_undecided(lazy):
    """Windows no decisive record decides (the C2 records K1 passes to the
    address check, codes 0 / 9 / 10, x 8): every window's extents evaluated --
    lazily from the tables, or, after the first call finds most windows
    undecided, by the extents module -- against the oracle, both modes."""
    import paper_2410_23661_b200 as pk
    from tracegen import workloads
    s, rec, args, meta = workloads.make_c2()
    codes = np.array(O.oracle_batch(s, rec, args), np.uint8)
    sub = rec[np.isin(codes, [0, 9, 10])]
    sub = sub[: len(sub) // 32 * 32]
    R = 8
    rec_t, args_t = workloads.replicate(sub, args, meta["ptr_mask"], R)
    p = pk.Picker(0, seq_lazy=lazy)
    p.load(s)
    for concurrent in (False, True, False):
        mode = O.SEQ_CONCURRENT if concurrent else O.SEQ_SEQUENTIAL
        want = np.tile(np.array(O.oracle_windows(s, sub, args, 32, mode), np.uint8), R)
        got = p.validate_sequence(rec_t, args_t, 32, concurrent=concurrent).cpu().numpy()
        assert p.last_launch_count() == 1
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, (concurrent, bad[:8], got[bad[:8]])
        assert (want == 0).sum() > 0 and (want == 10).sum() > 0
