"""Seeded inputs at the edges of the specialised module's code generation
(tests/test_gpu_codegen.py, tests/test_codegen_cpu.py).

Inputs only: summaries with coefficients at the int32 boundary, argument-valued
coefficients, gidx terms, and precondition bounds beyond / at the operands' type
ranges; records with values on both sides of every bound and pointers placed
near the far end of the read extents.  No verdict is computed here: expected
codes come from oracle/."""
import numpy as np

from .golden import desc, kernel, term
from .records import RecordBuilder

PTR_HI = (1 << 56) - 1
I31 = 1 << 31


def edge_summary():
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


def edge_records(seed, n=4000):
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
