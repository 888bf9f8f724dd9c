"""One picker_validate_models call on C2 x686 (for ncu: the fused kernel is
the second k_validate_pipe launch; the first is a warm-up)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_23661_b200 as pk  # noqa: E402
from tracegen import workloads  # noqa: E402

s, rec, args, meta = workloads.make_c2()
p = pk.Picker(0)
p.load(s)
rd, ad = p.replicate(rec, args, meta["ptr_mask"], 686)
n = rd.shape[0]
ctx = torch.from_numpy((np.arange(n, dtype=np.int64) % 97 + 1) * 4096).cuda()
for _ in range(2):
    (f, _, _), m = p.validate_models(rd, ad, ctx)
torch.cuda.synchronize()
print(m["n_idem"], m["unknown_input"])
