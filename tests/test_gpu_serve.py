"""The resident validator (picker_serve_*): one warp polling a mapped host
mailbox answers per-launch requests with the same codes as the oracle, and its
host-observed latency is measured (the paper's per-launch use)."""
import time

import numpy as np
import pytest

import oracle.picker_oracle as O
from tracegen import golden, workloads
from tracegen.records import RecordBuilder
from tracegen.synth import random_records, random_summary

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    import paper_2410_23661_b200 as pk
    return pk


def _requests(rec, args, sizes, rng):
    """Split records into requests of the given sizes, each with its own
    relative argument block (arg_off rebased)."""
    i = 0
    while i < len(rec):
        m = int(sizes[int(rng.integers(0, len(sizes)))])
        sub = rec[i:i + m].copy()
        offs = sub["arg_off"].astype(np.int64)
        blocks = [args[o:o + int(n)] for o, n in zip(offs, sub["nargs"])]
        a = np.concatenate(blocks) if blocks else np.zeros(0, np.int64)
        sub["arg_off"] = np.concatenate([[0], np.cumsum([len(b) for b in blocks])[:-1]]).astype(np.uint64)
        yield i, sub, a
        i += m


@pytest.mark.parametrize("which", ["golden", "random", "c2"])
def test_serve_parity(pk, which):
    if which == "golden":
        s = golden.golden_summary()
        b = RecordBuilder()
        for a in golden.C1_ARGS:
            b.add(0, a, grid=(4,), block=(128,))
        rec, args = b.build()
    elif which == "random":
        s = random_summary(71, n_kernels=24)
        rec, args = random_records(72, s, 600, max_threads=64, max_grid=8)
    else:
        s, rec, args, _ = workloads.make_c2()
        rec = rec[:3000]
    want = np.array(O.oracle_batch(s, rec, args), np.uint8)
    p = pk.Picker(0, serve=1)
    p.load(s)
    p.serve_start()
    try:
        rng = np.random.default_rng(3)
        for i, sub, a in _requests(rec, args, [1, 2, 7, 32], rng):
            got = p.serve_validate(sub, a)
            assert np.array_equal(got, want[i:i + len(sub)]), (i, got, want[i:i + len(sub)])
    finally:
        p.serve_stop()
    # restart after stop, reload requires stop
    p.serve_start()
    with pytest.raises(pk.PickerError):
        p.load(s)
    p.serve_stop()
    p.close()


def test_serve_latency(pk):
    """Host-observed round trip of one-record requests (median of 2,000)."""
    s, rec, args, _ = workloads.make_c2()
    p = pk.Picker(0, serve=1)
    p.load(s)
    p.serve_start()
    reqs = list(_requests(rec[:2000], args, [1], np.random.default_rng(0)))
    out = np.empty(1, np.uint8)
    ts = []
    for _, sub, a in reqs:
        t0 = time.perf_counter()
        p.serve_validate(sub, a, out=out)
        ts.append(time.perf_counter() - t0)
    p.serve_stop()
    p.close()
    med = 1e6 * float(np.median(ts))
    print(f"resident validator, 1 record: p50 {med:.2f} us, p90 {1e6 * float(np.percentile(ts, 90)):.2f} us")
    assert med < 50
