"""Run the validation kernels once on small inputs for compute-sanitizer
(memcheck / racecheck / synccheck): the pipelined tiled kernel at 64-record
tiles with >= 2 tiles per CTA (so the restaging, the next tile's key pass and
mbarrier phases >= 2 run), with one and two argument buffers, the sorted
schedule (C4-like kernels), the exact verifier and the sequence windows.
Checks the codes against the oracle too.

    compute-sanitizer --tool racecheck python scripts/sanitize.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle.picker_oracle as O  # noqa: E402
import paper_2410_23661_b200 as pk  # noqa: E402
from tracegen import workloads  # noqa: E402
from tracegen.synth import random_records, random_summary  # noqa: E402

s = random_summary(61, n_kernels=20)
rec, args = random_records(62, s, 1500, max_threads=64, max_grid=4)
want = np.array(O.oracle_batch_mp(s, rec, args), np.uint8)
R = 14  # 21,000 records: 329 tiles of 64 on 148 CTAs
rr, aa = workloads.replicate(rec, args, np.zeros(len(args), bool), R, delta=0)
for opt in [dict(tile=64, threads=64, ctas=1, args_per_rec=4, arg_bufs=1),
            dict(tile=64, threads=64, ctas=1, args_per_rec=4, arg_bufs=2)]:
    p = pk.Picker(0, **opt)
    p.load(s)
    f, _, _ = p.validate(rr, aa)
    assert (f.cpu().numpy() == np.tile(want, R)).all(), opt
    p.close()
    print("pipe", opt, "ok", flush=True)
s4, r4, a4, m4 = workloads.make_c4(n=1024, n_kernels=8)
w4 = np.array(O.oracle_batch_mp(s4, r4, a4), np.uint8)
p = pk.Picker(0)
p.load(s4)
r4t, a4t = workloads.replicate(r4, a4, m4["ptr_mask"], 4)
f, _, _ = p.validate(r4t, a4t)
assert (f.cpu().numpy() == np.tile(w4, 4)).all()
print("sorted ok", flush=True)
p.close()
p = pk.Picker(0)
p.load(s)
e, _ = p.exact_check(rec[:300], args, max_points=1 << 12)
assert (e.cpu().numpy() == np.array(O.oracle_batch(s, rec[:300], args, O.oracle_exact, cap=1 << 12), np.uint8)).all()
q = p.validate_sequence(rec[:500], args, 8).cpu().numpy()
assert (q == np.array(O.oracle_windows(s, rec[:500], args, 8), np.uint8)).all()
print("exact + sequence ok", flush=True)
torch.cuda.synchronize()
# round 2, session 3: the K2 kernel (wide-only summary), the fused models and
# K1's extents for the windows (64-record tiles: many tiles per CTA)
sw, rw, aw, _ = workloads.make_wide(n=150)
ww = np.array(O.oracle_batch(sw, rw, aw), np.uint8)
p = pk.Picker(0)
p.load(sw)
f, _, _ = p.validate(rw, aw)
assert p.last_launch_count() == 1 and (f.cpu().numpy() == ww).all()
p.close()
print("K2 kernel ok", flush=True)
s2, r2, a2, _ = workloads.make_c2()
w2 = np.array(O.oracle_batch_mp(s2, r2, a2), np.uint8)
ctx = (np.arange(len(r2), dtype=np.uint64) % 97 + 1) * 4096
p = pk.Picker(0, tile=64, threads=64, ctas=1, args_per_rec=4, arg_bufs=1)
p.load(s2)
(f, _, _), m = p.validate_models(r2, a2, ctx)
assert p.last_launch_count() == 1 and (f.cpu().numpy() == w2).all()
assert m == O.oracle_models(s2, r2, a2, w2, ctx)
print("fused models ok", flush=True)
q = p.validate_sequence(r2, a2, 32).cpu().numpy()
assert p.last_launch_count() == 2
assert (q == np.array(O.oracle_windows(s2, r2, a2, 32), np.uint8)).all()
print("windows on K1 extents ok", flush=True)
p.close()
torch.cuda.synchronize()
