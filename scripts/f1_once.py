"""Two picker_validate_sequence calls on C2 x686 (for ncu: profile the second)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_23661_b200 as pk  # noqa: E402
from tracegen import workloads  # noqa: E402

conc = len(sys.argv) > 1 and sys.argv[1] == "concurrent"
s, rec, args, meta = workloads.make_c2()
p = pk.Picker(0)
p.load(s)
rd, ad = p.replicate(rec, args, meta["ptr_mask"], 686)
for _ in range(2):
    out = p.validate_sequence(rd, ad, 32, concurrent=conc)
torch.cuda.synchronize()
print(int((out.cpu() <= 1).sum()))
