"""GPU parity for the specialised module's code generation (jit.cpp) at the
edges its optimisations depend on, and for every staging geometry.

* 32x32->64 multiplies are emitted only for terms the loader proves int32
  (coefficient and variable value): coefficients at +-(2^31 - 1), +-2^31 and
  argument-valued coefficients, with grids at the launch limit.
* Preconditions on launch dimensions and i32 arguments are one 32-bit compare
  after clamping the bounds to the operand's type range: bounds beyond the type
  range, lo == hi, and values on both sides of every bound.
* Geometries: one / two argument buffers, tile sizes from 64 to 2048 records,
  spans that do not fit the staging buffer, unpacked arguments.

Expected codes always come from the oracle (oracle/picker_oracle.py)."""
import numpy as np
import pytest

import oracle.picker_oracle as O
from tracegen.golden import desc, kernel, term
from tracegen.records import RecordBuilder
from tracegen.synth import random_records, random_summary

pytestmark = pytest.mark.gpu

PTR_HI = (1 << 56) - 1
I31 = 1 << 31
JIT = dict(jit=1)
PATHS = [JIT, dict(jit=0, bucket=0)]


@pytest.fixture(scope="module")
def pk():
    import paper_2410_23661_b200 as pk
    return pk


def _codes(pk, summary, rec, args, packed=True, **opt):
    p = pk.Picker(0, **opt)
    p.load(summary)
    flags, _, _ = p.validate(rec, args, packed=packed)
    got = flags.cpu().numpy()
    p.close()
    return got


def _want(summary, rec, args):
    return np.array(O.oracle_batch_mp(summary, rec, args, O.oracle_interval), dtype=np.uint8)


def _assert_same(got, want):
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first at {bad[:8]}: gpu {got[bad[:8]]} oracle {want[bad[:8]]}"


def _edge_summary():
    ptr2 = [("p0", "ptr"), ("p1", "ptr"), ("s0", "i32")]
    pre = [{"op": "p0", "lo": 0, "hi": PTR_HI}, {"op": "p1", "lo": 0, "hi": PTR_HI},
           {"op": "s0", "lo": -I31, "hi": I31 - 1}, {"op": "gdim.x", "lo": 1, "hi": I31 - 1}]
    bid = {"bid.x": {"lo": [], "hi": []}}
    tid = {"tid.x": {"lo": [], "hi": []}}
    ks = []
    # coefficient k on bid.x (bid.x <= 2^31 - 2): int32 for |k| < 2^31 and k = -2^31
    for kid, k in enumerate([I31 - 1, I31, -I31, -I31 - 1, (1 << 32) - (1 << 27)]):
        ks.append(kernel(10 + kid, f"edge{kid}", ptr2,
                         [desc("R", 4, "p0", [term(k, (), "bid.x")], bid),
                          desc("W", 8, "p1", [term(1, (), "tid.x")], tid)], pre=pre))
    # argument-valued coefficients: s0 (int32 range) and 2 * s0 (not int32)
    ks.append(kernel(20, "argcoef1", ptr2,
                     [desc("R", 4, "p0", [term(1, ["s0"], "tid.x")], tid),
                      desc("W", 4, "p1", [term(4, (), "tid.x")], tid)], pre=pre))
    ks.append(kernel(21, "argcoef2", ptr2,
                     [desc("R", 4, "p0", [term(2, ["s0"], "tid.x")], tid),
                      desc("W", 4, "p1", [term(4, (), "tid.x")], tid)], pre=pre))
    # gidx.x up to gdim.x * bdim.x - 1 (2^41): never int32
    ks.append(kernel(22, "gidx", ptr2,
                     [desc("R", 4, "p0", [term(4, (), "gidx.x")], {"gidx.x": {"lo": [], "hi": []}}),
                      desc("W", 4, "p1", [term(4, (), "gidx.x")], {"gidx.x": {"lo": [], "hi": []}})],
                     pre=pre))
    # precondition / global-condition bounds beyond, at and inside the type ranges
    cparams = [("p0", "ptr"), ("s0", "i32"), ("s1", "i32"), ("s2", "i64"), ("s3", "i32")]
    cpre = [{"op": "p0", "lo": 0, "hi": PTR_HI},
            {"op": "s0", "lo": -(1 << 40), "hi": 1 << 40},
            {"op": "s1", "lo": 5, "hi": 5},
            {"op": "s2", "lo": -3, "hi": 1 << 40},
            {"op": "s3", "lo": -I31, "hi": -I31 + 2},
            {"op": "gdim.x", "lo": -5, "hi": 1 << 40},
            {"op": "gdim.y", "lo": 3, "hi": 70000},
            {"op": "bdim.x", "lo": 0, "hi": 2000},
            {"op": "bdim.z", "lo": 2, "hi": 2}]
    cglob = [{"op": "s0", "lo": -100, "hi": I31 - 1}, {"op": "gdim.z", "lo": 1, "hi": 1}]
    ks.append(kernel(30, "checks", cparams,
                     [desc("R", 4, "p0", [term(4, (), "tid.x")], tid),
                      desc("W", 4, "p0", [term(1, ["s2"]), term(4, (), "tid.x"), term(4096)], tid)],
                     pre=cpre, glob=cglob))
    return {"version": 1, "kernels": ks}


def _edge_records(seed, n=4000):
    rng = np.random.default_rng(seed)
    b = RecordBuilder()
    ids = [10, 11, 12, 13, 14, 20, 21, 22]
    gxs = [1, 2, 3, 1 << 20, I31 - 2, I31 - 1, I31, 0]
    bxs = [1, 2, 32, 1023, 1024, 1025]
    s0s = [-I31, -I31 + 1, -101, -100, -1, 0, 1, 7, I31 - 2, I31 - 1]
    for _ in range(n):
        if rng.random() < 0.25:  # the precondition kernel
            s0 = int(rng.choice(s0s)) | (int(rng.integers(0, 2)) << 40)  # junk above an i32 slot
            s1 = int(rng.choice([4, 5, 6, 5 + (1 << 32)]))
            s2 = int(rng.choice([-4, -3, 0, 4096, (1 << 40), (1 << 40) + 1]))
            s3 = int(rng.choice([-I31, -I31 + 2, -I31 + 3, I31 - 1]))
            grid = (int(rng.choice(gxs)), int(rng.choice([1, 2, 3, 65535, 0])), int(rng.choice([1, 2])))
            block = (int(rng.choice(bxs)), 1, int(rng.choice([1, 2, 3])))
            p0 = int(rng.integers(1 << 32, 1 << 44)) & ~15
            b.add(30, [p0, s0, s1, s2, s3], grid=grid, block=block)
            continue
        kid = int(rng.choice(ids))
        gx = int(rng.choice(gxs))
        bxv = int(rng.choice(bxs))
        s0 = int(rng.choice(s0s))
        p0 = int(rng.integers(1 << 40, 1 << 44)) & ~15
        # p1 near the far end of p0's extent (touching / overlapping / clear)
        k = {10: I31 - 1, 11: I31, 12: -I31, 13: -I31 - 1, 14: (1 << 32) - (1 << 27)}.get(kid, 4)
        reach = k * max(gx - 1, 0) if kid < 20 else (s0 * (bxv - 1) if kid < 22 else 4 * gx * bxv)
        d = int(rng.choice([-16, -8, -4, -1, 0, 1, 3, 4, 5, 64]))
        p1 = p0 + reach + d if rng.random() < 0.7 else p0 + d
        p1 = min(max(p1, 0), PTR_HI)
        b.add(kid, [p0, p1, s0], grid=(gx, 1, 1), block=(bxv, 1, 1))
    return b.build()


@pytest.mark.parametrize("opt", PATHS, ids=str)
@pytest.mark.parametrize("seed", [1, 2])
def test_codegen_edges(pk, opt, seed):
    s = _edge_summary()
    rec, args = _edge_records(seed)
    _assert_same(_codes(pk, s, rec, args, **opt), _want(s, rec, args))


GEOMETRIES = [
    dict(jit=1),  # auto: 448 / 224 / 4 CTAs / one argument buffer for these summaries
    dict(jit=1, tile=448, threads=224, ctas=3, args_per_rec=5, arg_bufs=2),
    dict(jit=1, tile=896, threads=448, ctas=2, args_per_rec=5, arg_bufs=1),
    dict(jit=1, tile=2048, threads=512, ctas=1, args_per_rec=1, arg_bufs=1),
    dict(jit=1, tile=64, threads=32, ctas=8, args_per_rec=2, arg_bufs=1),  # spans overflow the buffer
    dict(jit=1, tile=64, threads=32, ctas=8, args_per_rec=2, arg_bufs=2),
]


@pytest.mark.parametrize("opt", GEOMETRIES, ids=str)
def test_geometries(pk, opt):
    s = random_summary(31, n_kernels=30)
    rec, args = random_records(32, s, 7001, max_threads=256, max_grid=32)  # ragged tail
    want = _want(s, rec, args)
    _assert_same(_codes(pk, s, rec, args, **opt), want)
    perm = np.random.default_rng(3).permutation(len(rec))  # arguments out of record order
    _assert_same(_codes(pk, s, rec[perm], args, packed=False, **opt), want[perm])


@pytest.mark.parametrize("opt", [dict(jit=1), dict(jit=1, wide_pairs=4), dict(jit=1, stride=1)], ids=str)
def test_small_batch_kernel(pk, opt):
    """n <= 1024 takes the one-CTA small-batch kernel (no staging, counts
    written instead of accumulated); around its limit the tiled kernel."""
    s = random_summary(41, n_kernels=30)
    rec, args = random_records(42, s, 1100, max_threads=256, max_grid=32)
    want_all = np.array(O.oracle_batch_mp(s, rec, args, O.oracle_interval, stride=bool(opt.get("stride"))),
                        dtype=np.uint8)
    p = pk.Picker(0, **opt)
    p.load(s)
    for n in (1, 31, 32, 33, 1000, 1024, 1025, 1100):
        flags, bits, counts = p.validate(rec[:n], args)
        want = want_all[:n]
        _assert_same(flags.cpu().numpy(), want)
        exp_c = np.zeros(16, np.int64)
        for c in want:
            exp_c[c if c <= 11 else 15] += 1
        assert np.array_equal(counts.cpu().numpy(), exp_c), n
        idem = np.pad((want <= 1).astype(np.uint8), (0, (-n) % 32)).reshape(-1, 32)[:, ::-1]
        assert np.array_equal(bits.cpu().numpy().view(np.uint32),
                              np.packbits(idem, axis=1).view(">u4").reshape(-1).astype(np.uint32)), n
    p.close()
