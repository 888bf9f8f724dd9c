"""Row f2 (Base / Base+R / Full breakdown, §7.4 l.1588-1611): the
"Base+R" input -- a summary WITHOUT range compaction.

Range compaction (§5.3, l.1029-1069) keeps a loop's induction variable
as a range variable so that an instruction inside a loop is one symbolic address
instead of one per unrolled iteration ("Our strawman solution unrolls the loop
and generates 32 symbolic addresses for this instruction", l.1062-1063).  This
module undoes it on a summary: a descriptor whose first induction variable
``ind*`` has one lower bound L becomes ``unroll`` descriptors, copy k < unroll-1
pinning the variable to L + k (its upper bounds kept, so a copy past the trip
count is empty) and the last copy covering [L + unroll - 1, hi].  The copies'
point sets partition the original one, so the result is a summary of the same
kernel with unroll x the symbolic addresses of that loop.

Input preparation only (summary -> summary): no range, overlap or verdict is
computed here.  Both the GPU path and the oracle consume the rewritten summary.
"""
from __future__ import annotations

import copy


def _shift(bexpr, k):
    e = copy.deepcopy(bexpr)
    e["k0"] = int(e["k0"]) + k
    return e


def uncompact_descriptor(d, unroll):
    """The copies of one descriptor (or [d] when it has no unrollable loop)."""
    var = next((v for v, spec in d["vars"].items()
                if v.startswith("ind") and len(spec.get("lo", [])) == 1 and "def" not in spec), None)
    if var is None or d.get("opaque"):
        return [d]
    spec = d["vars"][var]
    lo = spec["lo"][0]
    out = []
    for k in range(unroll):
        c = copy.deepcopy(d)
        s = c["vars"][var]
        s["lo"] = [_shift(lo, k)]
        if k < unroll - 1:
            s["hi"] = [_shift(lo, k)] + copy.deepcopy(spec.get("hi", []))
        out.append(c)
    return out


def uncompact(summary, unroll=32):
    """Base+R summary: every COND kernel's loop descriptors unrolled ``unroll``x."""
    out = copy.deepcopy(summary)
    for k in out["kernels"]:
        if k.get("class", "COND") != "COND":
            continue
        descs = []
        for d in k["desc"]:
            descs.extend(uncompact_descriptor(d, unroll))
        k["desc"] = descs
    return out
