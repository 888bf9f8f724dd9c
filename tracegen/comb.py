"""A "comb" kernel for the wide path's edge cases: nr read
sites A + 64 i + 4 j and nw write sites B + 64 i + 4 j (i the site, j < n an
induction variable), i.e. teeth of 4 n bytes every 64 bytes.  Depending on
B - A and n, write teeth fall between read teeth, touch them or overlap them.
Inputs only (no ranges or verdicts are computed here)."""
from __future__ import annotations

from .golden import bx, desc, kernel, ptr_pre, term


def comb_kernel(kid, nr, nw):
    v = {"ind0": {"lo": [bx(0)], "hi": [bx(-1, (1, ["n"]))]}}
    ds = [desc("R", 4, "A", [term(64 * i), term(4, (), "ind0")], v) for i in range(nr)]
    ds += [desc("W", 4, "B", [term(64 * i), term(4, (), "ind0")], v) for i in range(nw)]
    # interleave the kinds so descriptor order says nothing about lb order
    ds = [d for pair in zip(ds[:nr], ds[nr:]) for d in pair] + ds[min(nr, nw):nr] + ds[nr + min(nr, nw):]
    return kernel(kid, f"comb_{nr}x{nw}", [("A", "ptr"), ("B", "ptr"), ("n", "i64")], ds,
                  pre=ptr_pre("A", "B") + [{"op": "n", "lo": 0, "hi": 16}])


def comb_summary():
    """Kernel 0: 40 x 40 sites (80 descriptors: the smaller side sorted in the
    scratch); kernel 1: 600 x 500 sites (1,100 descriptors, still in the
    global scratch); kernel 2: 20 x 20 (40 descriptors: the register sort);
    kernel 3: 1500 x 1500 (beyond any scratch: lanes over pairs)."""
    return {"version": 1, "kernels": [comb_kernel(0, 40, 40), comb_kernel(1, 600, 500), comb_kernel(2, 20, 20),
                                      comb_kernel(3, 1500, 1500)]}
