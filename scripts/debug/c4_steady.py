"""Debug aid: run one C4 steady-state configuration (argv: R tile threads ctas args_per_rec|auto)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from tracegen import workloads
import paper_2410_23661_b200 as pk
R = int(sys.argv[1])
opt = dict(jit=1)
if len(sys.argv) > 2 and sys.argv[2] != "auto":
    t, th, c, a = map(int, sys.argv[2:6])
    opt.update(tile=t, threads=th, ctas=c, args_per_rec=a)
n = int(os.environ.get("C4_N", 1 << 12))
s, rec, args, meta = workloads.make_c4(n=n)
rec_t, args_t = workloads.replicate(rec, args, meta["ptr_mask"], R)
p = pk.Picker(0, **opt)
p.load(s)
f, b, c = p.validate(rec_t, args_t)
torch.cuda.synchronize()
print("ok", R, opt, n, np.bincount(f.cpu().numpy()))
