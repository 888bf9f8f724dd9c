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
from tracegen.edges import edge_records, edge_summary
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


@pytest.mark.parametrize("opt", PATHS, ids=str)
@pytest.mark.parametrize("seed", [1, 2])
def test_codegen_edges(pk, opt, seed):
    s = edge_summary()
    rec, args = edge_records(seed)
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
