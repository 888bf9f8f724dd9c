"""Row f2 (Base / Base+R / Full, §7.4 l.1588-1611): pins for the
uncompacted (Base+R) summary and GPU parity of the three versions' verdicts.

Base+R's summary comes from tracegen.uncompact (input preparation); both sides
consume it.  Pins: the copies' point sets partition the original descriptor's
(brute force), and the refinement chain exact NI => Base+R NI => Full NI."""
import numpy as np
import pytest

import oracle.picker_oracle as O
from tracegen import golden, workloads
from tracegen.records import RecordBuilder
from tracegen.synth import random_records, random_summary
from tracegen.uncompact import uncompact, uncompact_descriptor


def _batch(seed, n=250):
    s = random_summary(seed, n_kernels=12)
    rec, args = random_records(seed + 1000, s, n, max_threads=24, max_grid=3)
    return s, rec, args


@pytest.mark.parametrize("seed", [71, 72])
@pytest.mark.parametrize("unroll", [2, 3, 32])
def test_copies_partition_the_points(seed, unroll):
    """For every active descriptor with a loop, the multiset union of its
    copies' enumerated points equals its own points (no loss, no double count)."""
    s, rec, args = _batch(seed, n=120)
    K = O.index_summary(s)
    checked = 0
    for row in rec:
        r = O.decode_record(row, args)
        code, st = O._prefix(K, r)
        if code is not None:
            continue
        _, vals, active = st
        for d, box in active:
            copies = uncompact_descriptor(d, unroll)
            if len(copies) == 1 or d["opaque"] or O._box_points(box) > 4096:
                continue
            want = sorted(tuple(sorted(p.items())) for p in O._points(d, box))
            got = []
            for c in copies:
                cb = O.var_box(c, vals)
                if any(lo > hi for lo, hi in cb.values()):
                    continue
                got.extend(tuple(sorted(p.items())) for p in O._points(c, cb))
            assert sorted(got) == want
            checked += 1
    assert checked > 10


def test_relu_unrolled_32():
    """Fig. 4's relu: one read and one write descriptor over i in [0, N-1]
    (N <= 32 by the global condition) become 32 + 32 descriptors, as the
    strawman's unrolled loop ("generates 32 symbolic
    addresses for this instruction")."""
    s = golden.golden_summary()
    u = uncompact(s, 32)
    relu = next(k for k in u["kernels"] if k["id"] == 3)
    assert len(relu["desc"]) == 64


@pytest.mark.parametrize("seed", [73, 74, 75])
def test_refinement_chain(seed):
    """exact NI => Base+R NI => Full NI; only 10 -> 0 changes between them."""
    s, rec, args = _batch(seed)
    K, U = O.index_summary(s), O.index_summary(uncompact(s, 32))
    changed = 0
    for row in rec:
        r = O.decode_record(row, args)
        cf, cu = O.oracle_interval(K, r), O.oracle_interval(U, r)
        ce = O.oracle_exact(K, r, cap=1 << 13)
        if cf != cu:
            assert (cf, cu) == (O.NI_OVERLAP, O.IDEM_CHECKED)
            changed += 1
        if ce == O.NI_OVERLAP:
            assert cu == O.NI_OVERLAP


# ---- GPU: the three versions against the oracle ------------------------------

def _gpu(summary, rec, args):
    import paper_2410_23661_b200 as pk
    p = pk.Picker(0)
    p.load(summary)
    return p


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [76, 77])
def test_gpu_base_r_random(seed):
    s = random_summary(seed, n_kernels=30)
    rec, args = random_records(seed + 1000, s, 2000, max_threads=128, max_grid=16)
    u = uncompact(s, 32)
    flags, _, _ = _gpu(u, rec, args).validate(rec, args)
    want = np.array(O.oracle_batch_mp(u, rec, args), np.uint8)
    assert np.array_equal(flags.cpu().numpy(), want)


@pytest.mark.gpu
def test_gpu_three_versions_c3_small():
    """The breakdown workload (scripts/breakdown.py): Full = oracle_interval,
    Base+R = oracle_interval on the uncompacted summary, Base = oracle_exact."""
    s, rec, args, _ = workloads.make_c3(seed=23664, n=256, n_kernels=32, small=True)
    u = uncompact(s, 32)
    full, _, _ = _gpu(s, rec, args).validate(rec, args)
    base_r, _, _ = _gpu(u, rec, args).validate(rec, args)
    base, _ = _gpu(s, rec, args).exact_check(rec, args, max_points=1 << 24)
    assert np.array_equal(full.cpu().numpy(), np.array(O.oracle_batch_mp(s, rec, args), np.uint8))
    assert np.array_equal(base_r.cpu().numpy(), np.array(O.oracle_batch_mp(u, rec, args), np.uint8))
    want_exact = np.array(O.oracle_batch_mp(s, rec, args, O.oracle_exact, cap=1 << 24), np.uint8)
    assert np.array_equal(base.cpu().numpy(), want_exact)
