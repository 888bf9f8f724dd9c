"""Seeded random summaries and launch records for parity tests.

Inputs only: these functions choose summary shapes and argument values; they never
compute an address range, an overlap or a verdict.  The expected codes always come
from oracle/ (or from the paper, tests/golden/).

``random_summary`` produces kernels in the IR of DESIGN.md §3 that exercise every
feature the hot path supports: 1-D/2-D/3-D thread variables (tid/bid or gidx),
induction variables with argument-dependent trip counts, fresh variables with a
``mod``/``and`` definition, path-condition tightenings, floor-division terms,
negative (decreasing) coefficients, guards, opaque descriptors, global conditions
and kernel-level classes.  Preconditions bound every operand so that the summaries
are wrap-free (the loader checks this).
"""
from __future__ import annotations

import numpy as np

from .golden import bx, desc, kernel, term
from .records import RecordBuilder

PTR_HI = (1 << 56) - 1
WIDTHS = (1, 2, 4, 8, 16)
REASONS = ("SO", "ATOMIC", "IF", "PE", "NA")


def _scalar_names(k):
    return [p["name"] for p in k["params"] if p["kind"] != "ptr"]


def _ptr_names(k):
    return [p["name"] for p in k["params"] if p["kind"] == "ptr"]


def random_kernel(rng, kid, *, max_desc=8, max_dim=3, small=True):
    """One random kernel summary.  ``small`` keeps precondition boxes small enough
    that the exact (enumerating) oracle stays fast."""
    nptr = int(rng.integers(1, 6))
    nsc = int(rng.integers(0, 4))
    params = [(f"p{i}", "ptr") for i in range(nptr)]
    params += [(f"s{i}", "i32" if rng.random() < 0.6 else "i64") for i in range(nsc)]
    scal = [n for n, _ in params[nptr:]]
    pre = [{"op": n, "lo": 0, "hi": PTR_HI} for n, _ in params[:nptr]]
    s_hi = {}
    for n in scal:
        hi = int(rng.choice([8, 16, 64, 1024])) if small else int(rng.choice([64, 4096, 1 << 16]))
        lo = 0 if rng.random() < 0.85 else -int(rng.integers(1, 8))
        pre.append({"op": n, "lo": lo, "hi": hi})
        s_hi[n] = hi
    dims_hi = 64 if small else 65535
    pre.append({"op": "gdim.x", "lo": 1, "hi": dims_hi if small else (1 << 20)})
    pre.append({"op": "gdim.y", "lo": 1, "hi": 16 if small else 1024})
    glob = []
    if scal and rng.random() < 0.3:
        n = str(rng.choice(scal))
        glob.append({"op": n, "lo": -(1 << 63), "hi": int(rng.integers(1, s_hi[n] + 1))})

    ndim = int(rng.integers(1, max_dim + 1))
    axes = "xyz"[:ndim]
    descs = []
    nd = int(rng.integers(1, max_desc + 1))
    for _ in range(nd):
        kind = "R" if rng.random() < 0.55 else "W"
        width = int(rng.choice(WIDTHS))
        opaque = rng.random() < 0.04
        base = None if (opaque and rng.random() < 0.5) else str(rng.choice([n for n, _ in params[:nptr]]))
        vars_, terms = {}, []
        use_gidx = rng.random() < 0.5
        for a in axes:
            if rng.random() < 0.25 and a != "x":
                continue
            names = [f"gidx.{a}"] if use_gidx else [f"bid.{a}", f"tid.{a}"]
            for v in names:
                spec = {"lo": [], "hi": []}
                if scal and rng.random() < 0.2:  # tightening "v < s" -> hi = s - 1
                    spec["hi"].append(bx(-1, (1, [str(rng.choice(scal))])))
                if rng.random() < 0.1:  # lower tightening "v >= c"
                    spec["lo"].append(bx(int(rng.integers(0, 4))))
                vars_[v] = spec
        if scal and rng.random() < 0.4:  # induction counter i in [0, s-1]
            s = str(rng.choice(scal))
            vars_["ind0"] = {"lo": [bx(0)], "hi": [bx(-1, (1, [s]))]}
        if rng.random() < 0.2:  # fresh var from a periodic subexpression
            src = str(rng.choice(list(vars_))) if vars_ else None
            if src is not None and not src.startswith("fr"):
                if rng.random() < 0.5:
                    m = int(rng.integers(2, 12))
                    vars_["fr0"] = {"lo": [bx(0)], "hi": [bx(m - 1 + int(rng.integers(0, 2)))],
                                    "def": {"src": src, "mod": m}}
                else:
                    mask = int(rng.choice([1, 3, 7, 15]))
                    vars_["fr0"] = {"lo": [bx(0)], "hi": [bx(mask)], "def": {"src": src, "and": mask}}
        for v in list(vars_):
            if rng.random() < 0.15:
                continue  # a variable that only shapes the box (e.g. a def source)
            sign = -1 if rng.random() < 0.1 else 1
            for _ in range(int(rng.integers(1, 3))):
                k = sign * int(rng.choice([1, 2, 4, 8, 16]))
                f = []
                r = rng.random()
                if r < 0.3 and scal:
                    f = [str(rng.choice(scal))]
                    if pre[[p["op"] for p in pre].index(f[0])]["lo"] < 0:
                        f = []  # keep coefficient signs definite
                elif r < 0.5:
                    f = [f"bdim.{axes[0]}"]
                div = int(rng.choice([1, 1, 1, 2, 3, 8]))
                terms.append(term(k, f, v, div))
        if rng.random() < 0.3:
            terms.append(term(int(rng.integers(-64, 65)), [], None))
        guard = []
        if rng.random() < 0.15:
            a = str(rng.choice(scal)) if scal else "bdim.x"
            guard.append({"a": a, "cmp": str(rng.choice(["<", "<=", ">", ">=", "==", "!="])),
                          "b": int(rng.integers(0, 16)) if rng.random() < 0.7 else "gdim.x"})
        descs.append(desc(kind, width, base, terms if not opaque else [], vars_, guard, opaque))
    cls, reason = "COND", None
    r = rng.random()
    if r < 0.05:
        cls = "IDEM"  # write-only kernel
        for d in descs:
            d["kind"] = "W"
    elif r < 0.12:
        cls, reason = "NONIDEM", str(rng.choice(REASONS))
    return kernel(kid, f"rk{kid}", params, descs, pre=pre, glob=glob, cls=cls, reason=reason)


def random_summary(seed, n_kernels=16, **kw):
    rng = np.random.default_rng(seed)
    return {"version": 1, "kernels": [random_kernel(rng, i, **kw) for i in range(n_kernels)]}


def random_records(seed, summary, n, *, max_threads=64, max_grid=4, faults=True):
    """Random launch records for ``summary``'s kernels.

    Pointers are either spread far apart (distinct allocations) or packed within a
    few KB (so that extents touch and overlap), and sometimes aliased outright (the
    paper's way of generating non-idempotent instances).
    """
    rng = np.random.default_rng(seed)
    ks = summary["kernels"]
    b = RecordBuilder()
    for _ in range(n):
        k = ks[int(rng.integers(0, len(ks)))]
        kid = k["id"]
        pre = {c["op"]: (c["lo"], c["hi"]) for c in k["pre"]}
        bdim = [int(rng.integers(1, max_threads + 1)), 1, 1]
        if rng.random() < 0.3:
            bdim[1] = int(rng.integers(1, 5))
        if rng.random() < 0.15:
            bdim[2] = int(rng.integers(1, 3))
        gdim = [int(rng.integers(1, max_grid + 1)), 1, 1]
        if rng.random() < 0.3:
            gdim[1] = int(rng.integers(1, 3))
        if rng.random() < 0.1:
            gdim[2] = int(rng.integers(1, 3))
        close = rng.random() < 0.6
        region = int(rng.integers(1 << 20, 1 << 40)) & ~0xFF
        args = []
        ptrs = []
        for p in k["params"]:
            if p["kind"] == "ptr":
                if ptrs and rng.random() < 0.12:
                    v = int(rng.choice(ptrs))  # alias
                elif close:
                    v = region + int(rng.integers(0, 64)) * int(rng.choice([1, 4, 16, 64]))
                else:
                    v = region + int(rng.integers(0, 1 << 12)) * (1 << 24)
                ptrs.append(v)
            else:
                lo, hi = pre.get(p["name"], (0, 64))
                v = int(rng.integers(lo, hi + 1))
                if faults and rng.random() < 0.03:
                    v = hi + 1  # precondition violation
                if p["kind"] == "i32" and rng.random() < 0.02:
                    v |= 0x5A5A << 40  # junk in the upper half of an i32 slot
            args.append(v)
        if faults and rng.random() < 0.02 and ptrs:
            args[0] = 1 << 57  # pointer precondition violation
        nargs = None
        if faults and rng.random() < 0.01:
            nargs = len(args) + 1
        if faults and rng.random() < 0.01:
            kid = 10_000 + int(rng.integers(0, 10))
        if faults and rng.random() < 0.01:
            bdim[0] = 2048
        b.add(kid, args, grid=gdim, block=bdim, nargs=nargs)
    return b.build()
