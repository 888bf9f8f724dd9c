"""Instance-level verdict mix of the synthetic C2 trace, per app, from the
ORACLE (used to calibrate tracegen.workloads.KNOBS against PAPER.md Table 3)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle.picker_oracle as O  # noqa: E402
from tracegen.workloads import APPS, make_c2  # noqa: E402

PAPER_PICKER_NI = {"Rodinia": 494, "Parboil": 811, "TVM": 13, "PyTorch": 746, "TensorRT": 211, "FT": 4197}

t = time.time()
s, rec, args, meta = make_c2()
print(f"generated {len(rec)} records, {len(s['kernels'])} kernels, {len(args)} arg slots "
      f"({(len(rec) * 32 + len(args) * 8) / len(rec):.1f} B/record) in {time.time() - t:.1f}s")
t = time.time()
codes = np.array(O.oracle_batch_mp(s, rec, args), np.uint8)
print(f"oracle: {time.time() - t:.1f}s")
for ai, (app, nk, ninst, *_) in enumerate(APPS):
    c = codes[meta["app"] == ai]
    ni = int((c > 1).sum())
    hist = {int(k): int(v) for k, v in zip(*np.unique(c, return_counts=True))}
    print(f"{app:9s} n={len(c):6d} I={len(c) - ni:6d} NI={ni:6d} (paper Picker NI {PAPER_PICKER_NI[app]:5d}) {hist}")
ni = int((codes > 1).sum())
print(f"ALL       n={len(codes)} I={len(codes) - ni} NI={ni} (paper 11,745 / 6,472)")
