"""Experiment: throughput of the validation kernel on a trace in record order
vs the same records sorted by kernel id (what a global shape pre-sort would
give each tile).  Codes are checked to be the same multiset per kernel."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2410_23661_b200 as pk
from tracegen import workloads

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c4")
ap.add_argument("--replicas", type=int, default=512)
ap.add_argument("--opt", action="append", default=[])
ap.add_argument("--only", default=None, choices=[None, "record_order", "sorted_by_kernel"])
a = ap.parse_args()
make = {"c2": workloads.make_c2, "c3": workloads.make_c3, "c4": lambda: workloads.make_c4(n=1 << 13),
        "wide": workloads.make_wide}[a.workload]
s, rec, args, meta = make()
rr, aa = workloads.replicate(rec, args, meta["ptr_mask"], a.replicas)
opts = {k: int(v) for k, v in (kv.split("=") for kv in a.opt)}
p = pk.Picker(0, **opts)
p.load(s)
out = {}
for name, order in [("record_order", None), ("sorted_by_kernel", np.argsort(rr["kernel_id"], kind="stable"))]:
    if a.only and name != a.only:
        continue
    r = rr if order is None else rr[order]
    rd = torch.from_numpy(r.view(np.uint8).reshape(-1, 32)).cuda()
    ad = torch.from_numpy(aa).cuda()
    n = len(r)
    f = torch.empty(n, dtype=torch.uint8, device="cuda")
    b = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
    c = torch.empty(16, dtype=torch.int64, device="cuda")
    for _ in range(3):
        p.validate(rd, ad, out=(f, b, c), packed=order is None)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        p.validate(rd, ad, out=(f, b, c), packed=order is None)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    out[name] = {"ms": ms, "G_inst_s": n / ms / 1e6, "counts": c.cpu().tolist()}
print(json.dumps(out))
