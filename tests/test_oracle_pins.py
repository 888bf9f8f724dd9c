"""Pins for the CPU oracle: paper values, brute-force kernel
simulations written from the kernels' source semantics (not from the summary IR),
closed forms and invariants.  CPU only."""
import json
import os

import numpy as np
import pytest

import oracle.picker_oracle as O
from tracegen import golden
from tracegen.records import RecordBuilder
from tracegen.synth import random_records, random_summary

HERE = os.path.dirname(__file__)


def _rec(kid, args, grid=(1, 1, 1), block=(1, 1, 1), nargs=None):
    b = RecordBuilder()
    b.add(kid, args, grid=grid, block=block, nargs=nargs)
    rec, pool = b.build()
    return O.decode_record(rec[0], pool)


@pytest.fixture(scope="module")
def G():
    return O.index_summary(golden.golden_summary())


def _cases():
    with open(os.path.join(HERE, "golden", "paper_examples.json")) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c["name"])
def test_paper_examples(G, case):
    r = _rec(case["kernel_id"], case["args"], case["grid"], case["block"])
    assert O.oracle_interval(G, r) == case["interval"]
    assert O.oracle_interval(G, r, stride=True) == case.get("stride", case["interval"])
    assert O.oracle_exact(G, r) == case["exact"]
    if "extents" in case:
        code, ext = O.extents(G, r)
        assert code is None
        assert sorted(map(tuple, case["extents"])) == sorted(ext)


# ---- brute-force kernel simulations (the kernels' code, PAPER Fig. 1 / Fig. 4) ----

def sim_vector_add(A, B, C, g, b):
    R, W = set(), set()
    for bid in range(g):
        for tid in range(b):
            idx = bid * b + tid
            R.update(range(B + 4 * idx, B + 4 * idx + 4))
            R.update(range(C + 4 * idx, C + 4 * idx + 4))
            W.update(range(A + 4 * idx, A + 4 * idx + 4))
    return R, W


def sim_relu(A, B, N, g, b):
    R, W = set(), set()
    for bid in range(g):
        for tid in range(b):
            for i in range(N):
                e = (bid * b + tid) * N + i
                R.update(range(A + 4 * e, A + 4 * e + 4))
                W.update(range(B + 4 * e, B + 4 * e + 4))
    return R, W


def sim_tighten(A, B, N, b):
    R, W = set(), set()
    for tid in range(b):
        if tid < N:
            R.update(range(A + 4 * tid, A + 4 * tid + 4))
            W.update(range(B + 4 * tid, B + 4 * tid + 4))
    return R, W


def sim_modfresh(A, B, b):
    R, W = set(), set()
    for tid in range(b):
        R.update(range(A + 4 * (tid % 10), A + 4 * (tid % 10) + 4))
        W.update(range(B + 4 * tid, B + 4 * tid + 4))
    return R, W


def _check_against_sim(G, kid, args, grid, block, R, W):
    r = _rec(kid, args, (grid, 1, 1), (block, 1, 1))
    code_i = O.oracle_interval(G, r)
    code_e = O.oracle_exact(G, r)
    truth = 10 if R & W else 0
    assert code_e == truth
    # no false positives: interval says idempotent => truly idempotent
    if code_i == 0:
        assert truth == 0
    # each extent covers its site and is tight (LB = min over threads, l.933-935)
    _, ext = O.extents(G, r)
    rex = [(lb, ub) for k, lb, ub in ext if k == "R"]
    wex = [(lb, ub) for k, lb, ub in ext if k == "W"]
    for s, ex in ((R, rex), (W, wex)):
        for x in s:
            assert any(lb <= x <= ub for lb, ub in ex)
    return code_i, code_e


def test_sim_vector_add(G):
    rng = np.random.default_rng(1)
    for _ in range(60):
        g, b = int(rng.integers(1, 4)), int(rng.integers(1, 40))
        ptrs = [0x10000 + int(rng.integers(0, 64)) * 16 for _ in range(3)]
        R, W = sim_vector_add(*ptrs, g, b)
        ci, ce = _check_against_sim(G, 0, ptrs, g, b, R, W)
        assert ci == ce  # contiguous accesses: no range overestimation
        _, ext = O.extents(G, _rec(0, ptrs, (g, 1, 1), (b, 1, 1)))
        assert ("W", min(W), max(W)) in ext


def test_sim_relu_closed_form(G):
    """G4: read extent = [A, A + 4*gdim*bdim*N - 1]."""
    rng = np.random.default_rng(2)
    for _ in range(40):
        g, b, N = int(rng.integers(1, 4)), int(rng.integers(1, 17)), int(rng.integers(1, 9))
        A = 0x40000 + int(rng.integers(0, 32)) * 4
        B = A + int(rng.integers(-200, 200)) * 4
        R, W = sim_relu(A, B, N, g, b)
        ci, ce = _check_against_sim(G, 3, [A, B, N], g, b, R, W)
        assert ci == ce
        _, ext = O.extents(G, _rec(3, [A, B, N], (g, 1, 1), (b, 1, 1)))
        assert ("R", A, A + 4 * g * b * N - 1) in ext
        assert (min(R), max(R)) == (A, A + 4 * g * b * N - 1)


def test_sim_tighten(G):
    rng = np.random.default_rng(3)
    for _ in range(60):
        b, N = int(rng.integers(1, 40)), int(rng.integers(0, 50))
        A = 0x1000
        B = A + int(rng.integers(-40, 200))
        R, W = sim_tighten(A, B, N, b)
        ci, ce = _check_against_sim(G, 5, [A, B, N], 1, b, R, W)
        assert ci == ce
        if R:
            _, ext = O.extents(G, _rec(5, [A, B, N], (1, 1, 1), (b, 1, 1)))
            assert ("R", min(R), max(R)) in ext  # [0, min(N-1, bdim-1)], l.1025


def test_sim_modfresh(G):
    rng = np.random.default_rng(4)
    seen_ro = False
    for _ in range(80):
        b = int(rng.integers(1, 24))
        A = 0x1000
        B = A + int(rng.integers(-10, 60)) * 4
        R, W = sim_modfresh(A, B, b)
        ci, ce = _check_against_sim(G, 6, [A, B], 1, b, R, W)
        seen_ro |= (ci == 10 and ce == 0)
    assert seen_ro  # the fresh-variable rewrite over-approximates (l.992-993)


def test_stride_ro_sets(G):
    """PAPER l.1174-1177 literally: read {1,3,5}, write {0,2,4}."""
    r = _rec(4, [0], (1, 1, 1), (3, 1, 1))
    _, ext = O.extents(G, r)
    assert sorted(ext) == [("R", 1, 5), ("W", 0, 4)]
    assert O.oracle_interval(G, r) == 10 and O.oracle_exact(G, r) == 0


# ---- random summaries: invariants ---------------------------------------------

def _random_batch(seed, n=300):
    s = random_summary(seed, n_kernels=12)
    rec, args = random_records(seed + 1000, s, n, max_threads=24, max_grid=3)
    return s, O.index_summary(s), rec, args


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_interval_vs_exact(seed):
    """G12: interval = I => exact = I; exact = 10 => interval = 10; the only
    differences are interval 10 / exact 0 (range overestimation) or skips."""
    s, K, rec, args = _random_batch(seed)
    stats = {"same": 0, "ro": 0, "skip": 0}
    for row in rec:
        r = O.decode_record(row, args)
        ci = O.oracle_interval(K, r)
        ce = O.oracle_exact(K, r, cap=1 << 13)
        if ce == O.EXACT_SKIPPED:
            stats["skip"] += 1
            continue
        if ci == ce:
            stats["same"] += 1
        else:
            assert (ci, ce) == (10, 0), (ci, ce)
            stats["ro"] += 1
    assert stats["same"] > 100


@pytest.mark.parametrize("seed", [21, 22])
def test_exact_bytes_inside_extents(seed):
    """Range soundness: every enumerated byte lies in its descriptor's extent."""
    s, K, rec, args = _random_batch(seed, n=150)
    checked = 0
    for row in rec:
        r = O.decode_record(row, args)
        code, st = O._prefix(K, r)
        if code is not None:
            continue
        _, vals, active = st
        for d, box in active:
            if d["opaque"]:
                continue
            free = {v: b for v, b in box.items() if "def" not in d["vars"][v]}
            if O._box_points(free) > 4096:
                continue
            lb, ub = O.interval_extent(d, vals, box)
            addrs = [O._addr(d, vals, p) for p in O._points(d, box)]
            assert lb <= min(addrs) and max(addrs) + d["width"] - 1 <= ub
            if all("def" not in spec for spec in d["vars"].values()):
                assert (lb, ub) == (min(addrs), max(addrs) + d["width"] - 1)  # tight
            checked += 1
    assert checked > 50


@pytest.mark.parametrize("seed", [31, 32])
def test_box_vs_per_variable(monkeypatch, seed):
    """Whole-box brute force and per-variable minima agree (separable sum)."""
    s, K, rec, args = _random_batch(seed, n=200)
    ref = []
    for row in rec:
        ref.append(O.extents(K, O.decode_record(row, args)))
    monkeypatch.setattr(O, "BRUTE_BOX_POINTS", 0)
    for row, want in zip(rec, ref):
        assert O.extents(K, O.decode_record(row, args)) == want
    monkeypatch.setattr(O, "BRUTE_VAR_POINTS", 0)  # endpoints only (monotone)
    for row, want in zip(rec, ref):
        assert O.extents(K, O.decode_record(row, args)) == want


@pytest.mark.parametrize("seed", [41])
def test_translation_invariance(seed):
    """G9: moving every pointer by the same delta keeps the verdict."""
    s, K, rec, args = _random_batch(seed, n=200)
    for row in rec:
        r = O.decode_record(row, args)
        k = K.get(r["kernel_id"])
        if k is None or r["nargs"] != len(k["params"]):
            continue
        a = list(args[r["arg_off"]: r["arg_off"] + r["nargs"]])
        ptr = [p["kind"] == "ptr" for p in k["params"]]
        if any(p and not (0 <= int(v) < (1 << 55)) for p, v in zip(ptr, a)):
            continue
        moved = [int(v) + (1 << 50) if p else int(v) for p, v in zip(ptr, a)]
        r2 = _rec(r["kernel_id"], moved, r["grid"], r["block"])
        assert O.oracle_interval(K, r2) == O.oracle_interval(K, r)


def test_monotone_grid_growth(G):
    """G14: with non-negative coefficients, growing the grid never clears an overlap."""
    for g in range(1, 6):
        r1 = _rec(0, [0x1000, 0x1000 + 4 * 128 * g - 4, 0x9000], (g, 1, 1), (128, 1, 1))
        assert O.oracle_interval(G, r1) == 10
        r2 = _rec(0, [0x1000, 0x1000 + 4 * 128 * g - 4, 0x9000], (g + 1, 1, 1), (128, 1, 1))
        assert O.oracle_interval(G, r2) == 10


def test_i32_sign_extension(G):
    """i32 arguments take the low 32 bits of their slot."""
    junk = (0x77 << 40) | 16
    r = _rec(3, [65536, 131072, junk], (4, 1, 1), (32, 1, 1))
    assert O.oracle_interval(G, r) == 0
    r = _rec(3, [65536, 131072, 0xFFFFFFFF], (4, 1, 1), (32, 1, 1))  # N = -1 < 0
    assert O.oracle_interval(G, r) == 7


# ---- exact verifier: point cap (code 11) and far-apart accesses ------------------
# Code 11 is "the point count exceeds the cap" (reading Q22); there is
# no limit on the span of the addresses.

def test_exact_point_cap_boundary(G):
    """vectorAdd, gdim 4 x bdim 128: 3 symbolic addresses x 512 threads = 1,536
    points (every thread of every symbolic address)."""
    r = _rec(0, [0x1000, 0x2000, 0x3000], (4, 1, 1), (128, 1, 1))
    assert O.exact_points(G, r) == 1536
    assert O.oracle_exact(G, r, cap=1535) == O.EXACT_SKIPPED
    assert O.oracle_exact(G, r, cap=1536) == O.IDEM_CHECKED
    r = _rec(0, [0x1000, 0x2000, 0x1000], (4, 1, 1), (128, 1, 1))  # C aliases A
    assert O.oracle_exact(G, r, cap=1535) == O.EXACT_SKIPPED
    assert O.oracle_exact(G, r, cap=1536) == O.NI_OVERLAP
    # the opaque rule is decided before any point is counted (§8C order)
    r = _rec(9, [0x1000, 0x2000, 1, 1], (1, 1, 1), (32, 1, 1))
    assert O.oracle_exact(G, r, cap=0) == O.NI_OPAQUE


def far_stride_summary():
    """k(int* A, long S, long off): v = A[S*tid/4]; A[(S*tid + off)/4] = v
    (byte addresses A + S*tid and A + S*tid + off, 4 bytes each)."""
    t = {"tid.x": {"lo": [], "hi": []}}
    return {"version": 1, "kernels": [golden.kernel(
        0, "far_stride", [("A", "ptr"), ("S", "i64"), ("off", "i64")],
        [golden.desc("R", 4, "A", [golden.term(1, ["S"], "tid.x")], t),
         golden.desc("W", 4, "A", [golden.term(1, ["S"], "tid.x"), golden.term(1, ["off"])], t)],
        pre=golden.ptr_pre("A") + [{"op": "S", "lo": 0, "hi": 1 << 40}, {"op": "off", "lo": 0, "hi": 64}])]}


@pytest.mark.parametrize("off,exact", [(4, O.IDEM_CHECKED), (2, O.NI_OVERLAP), (0, O.NI_OVERLAP)])
def test_exact_far_apart_accesses(off, exact):
    """S = 2^36, bdim 4: reads {A + k S .. + 3}, writes {A + k S + off .. + 3},
    k = 0..3.  The range extents [A, A + 3 S + 3] and [A + off, A + 3 S + off + 3]
    overlap (interval 10); the byte sets share bytes only
    when off < 4 (l.717-730).  The shared window spans ~3 x 2^36 bytes."""
    K = O.index_summary(far_stride_summary())
    r = _rec(0, [1 << 44, 1 << 36, off], (1, 1, 1), (4, 1, 1))
    assert O.oracle_interval(K, r) == O.NI_OVERLAP
    assert O.oracle_exact(K, r) == exact


# ---- many symbolic addresses (row a8, the wide path's inputs) ---------------------

@pytest.mark.parametrize("kid,nr,nw", [(0, 40, 40), (1, 600, 500), (2, 20, 20), (3, 1500, 1500)])
def test_comb_kernels(kid, nr, nw):
    """Read teeth [A + 64 i, A + 64 i + 4 n - 1], write teeth at B (hand-derived,
    closed byte intervals, PAPER.md l.658-666 and reading Q4):
    B = A + 64 nr, n = 16: the first write byte follows the last read byte -> 0;
    B = A + 64 (nr - 1), n = 1: write tooth 0 = read tooth nr - 1 -> 10;
    B = A + 32, n = 8: teeth interleave and touch -> 0; n = 9: 4 bytes shared -> 10;
    B = A - 64 nw: every write tooth below A -> 0; n = 0: no tooth -> 0."""
    from tracegen.comb import comb_summary
    K = O.index_summary(comb_summary())
    A = 1 << 40
    got = [O.oracle_interval(K, _rec(kid, [A, B, n], (1, 1, 1), (32, 1, 1)))
           for B, n in [(A + 64 * nr, 16), (A + 64 * (nr - 1), 1), (A + 32, 8), (A + 32, 9), (A - 64 * nw, 16),
                        (A, 0)]]
    assert got == [0, 10, 0, 10, 0, 0]
