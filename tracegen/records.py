"""Launch-record wire format and a packer for it.

This module is shared by the oracle side and the CUDA side *only as an input
generator*: it lays out bytes, it holds none of the validation arithmetic.

A launch record is a 32-byte little-endian header plus ``nargs`` 64-bit slots in
a shared ``int64`` argument pool (an instance = kernel identity + launch
arguments + grid/block dimensions, "an instance refers to the
invocation of a GPU kernel with a specific input state and arguments";
l.725-726 restricts the pseudocode to 1-D "without loss of generality", here
3-D with 1-D as y = z = 1).

    off  type      field
    0    u32       kernel_id
    4    u32       nargs
    8    u32       grid.x
    12   u16,u16   grid.y, grid.z
    16   u16 x4    block.x, block.y, block.z, reserved (0)
    24   u64       arg_off  (index into the int64 args pool)
"""
from __future__ import annotations

import numpy as np

REC_DTYPE = np.dtype(
    [
        ("kernel_id", "<u4"),
        ("nargs", "<u4"),
        ("grid_x", "<u4"),
        ("grid_y", "<u2"),
        ("grid_z", "<u2"),
        ("block_x", "<u2"),
        ("block_y", "<u2"),
        ("block_z", "<u2"),
        ("reserved", "<u2"),
        ("arg_off", "<u8"),
    ]
)
assert REC_DTYPE.itemsize == 32


def i64(v: int) -> int:
    """Store an unsigned 64-bit pattern (e.g. a pointer) in a signed slot."""
    v &= (1 << 64) - 1
    return v - (1 << 64) if v >= (1 << 63) else v


class RecordBuilder:
    """Accumulates launch records into a packed (args_packed=1) batch."""

    def __init__(self):
        self._rows = []
        self._args = []

    def add(self, kernel_id, args, grid=(1, 1, 1), block=(1, 1, 1), nargs=None):
        grid = tuple(grid) + (1,) * (3 - len(grid))
        block = tuple(block) + (1,) * (3 - len(block))
        off = len(self._args)
        self._args.extend(i64(int(a)) for a in args)
        self._rows.append(
            (
                kernel_id,
                len(args) if nargs is None else nargs,
                grid[0], grid[1], grid[2],
                block[0], block[1], block[2], 0,
                off,
            )
        )
        return len(self._rows) - 1

    def __len__(self):
        return len(self._rows)

    def build(self):
        rec = np.array(self._rows, dtype=REC_DTYPE) if self._rows else np.zeros(0, REC_DTYPE)
        args = np.array(self._args, dtype=np.int64) if self._args else np.zeros(0, np.int64)
        return rec, args


def concat(batches):
    """Concatenate (rec, args) batches, rebasing arg_off."""
    recs, argss, base = [], [], 0
    for rec, args in batches:
        r = rec.copy()
        r["arg_off"] += base
        recs.append(r)
        argss.append(args)
        base += len(args)
    return np.concatenate(recs), np.concatenate(argss)
