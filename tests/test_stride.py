"""Row f4 (stride-aware ranges, reading Q24): pins for the oracle's congruence
refinement and GPU parity of the library's stride mode.

Pins (none retypes the oracle's formula): the paper's RO example
(PAPER.md l.1174-1177), brute-force enumeration of the pair test over explicit
address sets, the gcd of enumerated address differences, and soundness against
the exact (enumerating) oracle on random summaries."""
import itertools
import math

import numpy as np
import pytest

import oracle.picker_oracle as O
from tracegen import golden
from tracegen.records import RecordBuilder
from tracegen.synth import random_records, random_summary


def _rec(kid, args, grid=(1, 1, 1), block=(1, 1, 1)):
    b = RecordBuilder()
    b.add(kid, args, grid=grid, block=block)
    rec, pool = b.build()
    return O.decode_record(rec[0], pool)


def test_paper_ro_example():
    """read {1,3,5} and write {0,2,4} do not overlap; the
    range model says they do, the stride-aware model recovers I."""
    G = O.index_summary(golden.golden_summary())
    r = _rec(4, [0], (1, 1, 1), (3, 1, 1))
    assert O.oracle_interval(G, r) == O.NI_OVERLAP
    assert O.oracle_interval(G, r, stride=True) == O.IDEM_CHECKED
    assert O.oracle_exact(G, r) == O.IDEM_CHECKED


@pytest.mark.parametrize("gr,gw", [(0, 0), (0, 3), (4, 0), (2, 2), (4, 6), (6, 9), (8, 12), (5, 7), (16, 16)])
def test_may_collide_brute_force(gr, gw):
    """The pair test equals an explicit search over the two progressions
    (widths 1..5, every residue pair): a in rR + gR*Z, b in rW + gW*Z, touching
    [a, a+wR-1] and [b, b+wW-1]."""
    span = 120
    for wr, ww in itertools.product(range(1, 6), repeat=2):
        for rr in (range(gr) if gr else range(-7, 8)):
            for rw in (range(gw) if gw else range(-7, 8)):
                A = [rr] if gr == 0 else range(rr - span * gr // max(gr, 1), span, gr)
                B = [rw] if gw == 0 else range(rw - span * gw // max(gw, 1), span, gw)
                Bs = set()
                for b in B:
                    Bs.update(range(b, b + ww))
                truth = any(x in Bs for a in A for x in range(a, a + wr))
                assert O.may_collide((gr, rr), wr, (gw, rw), ww) == truth, (gr, gw, rr, rw, wr, ww)


def _random_batch(seed, n=300):
    s = random_summary(seed, n_kernels=12)
    rec, args = random_records(seed + 1000, s, n, max_threads=24, max_grid=3)
    return s, O.index_summary(s), rec, args


@pytest.mark.parametrize("seed", [51, 52])
def test_congruence_is_gcd_of_address_differences(seed):
    """Every enumerated address is = r (mod g), and g is exactly the gcd of the
    differences of the enumerated addresses when every variable's terms share
    one divisor (descriptors without fresh definitions): a dropped or extra term
    changes g.  With mixed divisors g only divides that gcd."""
    s, K, rec, args = _random_batch(seed, n=150)
    checked = 0
    for row in rec:
        r = O.decode_record(row, args)
        code, st = O._prefix(K, r)
        if code is not None:
            continue
        _, vals, active = st
        for d, box in active:
            if d["opaque"] or any("def" in spec for spec in d["vars"].values()):
                continue
            if O._box_points(box) > 4096:
                continue
            addrs = [O._addr(d, vals, p) for p in O._points(d, box)]
            g, res = O.congruence(d, vals, box)
            diff_gcd = 0
            for a in addrs:
                diff_gcd = math.gcd(diff_gcd, abs(a - addrs[0]))
            divs = {}
            for t in d["terms"]:
                if t["var"] is not None:
                    divs.setdefault(t["var"], set()).add(t.get("div", 1))
            if all(len(v) == 1 for v in divs.values()):
                assert g == diff_gcd
            else:
                assert diff_gcd % g == 0 if g else diff_gcd == 0
            if g == 0:
                assert addrs == [res] * len(addrs)
            else:
                assert all(a % g == res for a in addrs)
            checked += 1
    assert checked > 50


@pytest.mark.parametrize("seed", [53, 54, 55])
def test_stride_between_interval_and_exact(seed):
    """Soundness and refinement: exact NI => stride NI => interval NI, and the
    stride variant never changes a code other than 10 -> 0."""
    s, K, rec, args = _random_batch(seed)
    same = 0
    for row in rec:
        r = O.decode_record(row, args)
        ci = O.oracle_interval(K, r)
        cs = O.oracle_interval(K, r, stride=True)
        ce = O.oracle_exact(K, r, cap=1 << 13)
        if ci != cs:
            assert (ci, cs) == (O.NI_OVERLAP, O.IDEM_CHECKED)
        if ce == O.NI_OVERLAP:
            assert cs == O.NI_OVERLAP
        same += ci == cs
    assert same > 100


def test_stride_recovers_ro_on_synthetic_traces():
    """The interleaved template of the C2 trace (reads even elements, writes odd
    ones) is the RO shape: the stride variant turns those records into I and the
    exact verifier agrees."""
    from tracegen import workloads
    s, rec, args, meta = workloads.make_c2()
    K = O.index_summary(s)
    rng = np.random.default_rng(7)
    idx = rng.choice(len(rec), size=1500, replace=False)
    recovered = 0
    for i in idx:
        r = O.decode_record(rec[i], args)
        ci = O.oracle_interval(K, r)
        cs = O.oracle_interval(K, r, stride=True)
        if ci != cs:
            recovered += 1
            assert O.oracle_exact(K, r, cap=1 << 16) in (O.IDEM_CHECKED, O.EXACT_SKIPPED)
    assert recovered > 0


# ---- GPU parity of the library's stride mode (picker_set_option "stride") -----

def _gpu_codes(summary, rec, args, at_load=False, **opt):
    """at_load: option set before picker_load_summaries (the specialised module
    is generated stride-aware); otherwise after it (table-driven stride path)."""
    import paper_2410_23661_b200 as pk
    p = pk.Picker(0, **opt)
    if at_load:
        p.set_option("stride", 1)
    p.load(summary)
    p.set_option("stride", 1)
    flags, bits, counts = p.validate(rec, args)
    return flags.cpu().numpy(), bits.cpu().numpy().view(np.uint32), counts.cpu().numpy()


def _want(summary, rec, args):
    return np.array(O.oracle_batch_mp(summary, rec, args, O.oracle_interval, stride=True), np.uint8)


def _check(got, want):
    flags, bits, counts = got
    bad = np.nonzero(flags != want)[0]
    assert bad.size == 0, f"{bad.size} mismatches at {bad[:8]}: gpu {flags[bad[:8]]} oracle {want[bad[:8]]}"
    n = len(want)
    idem = (want <= 1).astype(np.uint8)
    words = np.packbits(np.pad(idem, (0, (-n) % 32)).reshape(-1, 32)[:, ::-1], axis=1).view(">u4").reshape(-1)
    assert np.array_equal(bits, words.astype(np.uint32))
    exp = np.zeros(16, np.int64)
    for c in want:
        exp[c if c <= 11 else 15] += 1
    assert np.array_equal(counts, exp)


STRIDE_OPTS = [dict(jit=0), dict(jit=1), dict(jit=1, wide_pairs=4), dict(jit=1, at_load=True),
               dict(jit=1, wide_pairs=4, at_load=True)]


@pytest.mark.gpu
@pytest.mark.parametrize("opt", STRIDE_OPTS, ids=str)
def test_gpu_stride_paper_examples(opt):
    import json
    import os
    s = golden.golden_summary()
    cases = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))["cases"]
    b = RecordBuilder()
    for c in cases:
        b.add(c["kernel_id"], c["args"], c["grid"], c["block"])
    rec, args = b.build()
    want = np.array([c.get("stride", c["interval"]) for c in cases], np.uint8)
    _check(_gpu_codes(s, rec, args, **opt), want)


@pytest.mark.gpu
@pytest.mark.parametrize("at_load", [False, True])
@pytest.mark.parametrize("seed", [61, 62, 63])
def test_gpu_stride_random(seed, at_load):
    s = random_summary(seed, n_kernels=40)
    rec, args = random_records(seed + 1000, s, 3000, max_threads=256, max_grid=64)
    _check(_gpu_codes(s, rec, args, at_load=at_load), _want(s, rec, args))


@pytest.mark.gpu
@pytest.mark.parametrize("at_load", [False, True])
@pytest.mark.parametrize("which", ["c2", "c3"])
def test_gpu_stride_workloads(which, at_load):
    """The C2 trace (547 kernels) and the C3 base (64 kernels), every record
    against the oracle's stride variant; table-driven and specialised."""
    from tracegen import workloads
    s, rec, args, _ = workloads.make_c2() if which == "c2" else workloads.make_c3(n=1 << 12, n_kernels=64)
    _check(_gpu_codes(s, rec, args, at_load=at_load), _want(s, rec, args))


@pytest.mark.gpu
def test_gpu_stride_module_plain_verdicts():
    """A module generated stride-aware still answers plain (range-model)
    verdicts when the option is switched off after loading."""
    import paper_2410_23661_b200 as pk
    s = random_summary(64, n_kernels=30)
    rec, args = random_records(1064, s, 2000, max_threads=256, max_grid=64)
    p = pk.Picker(0)
    p.set_option("stride", 1)
    p.load(s)
    p.set_option("stride", 0)
    flags, _, _ = p.validate(rec, args)
    want = np.array(O.oracle_batch_mp(s, rec, args), np.uint8)
    assert np.array_equal(flags.cpu().numpy(), want)
