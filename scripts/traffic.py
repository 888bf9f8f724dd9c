"""DRAM traffic of one validate call per bench workload, for bench.py's
roofline.traffic (profiles/traffic.json).  Under ncu:

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:"k_validate|k_sort" \\
        --csv python scripts/traffic.py --workload c4 --calls 2

and `python scripts/traffic.py --collect out.csv --workload c4` sums the last call's kernels."""
import argparse
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--calls", type=int, default=2)
ap.add_argument("--collect", default=None)
ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "traffic.json"))
a = ap.parse_args()

import bench  # noqa: E402

if a.collect:
    lines = open(a.collect).read().splitlines()
    st = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(lines[st:]))
    h = rows[0]
    per = {}
    for r in rows[1:]:
        per.setdefault(int(r[h.index("ID")]), {"kernel": r[h.index("Kernel Name")].split("(")[0]})[
            r[h.index("Metric Name")]] = float(r[h.index("Metric Value")])
    ks = [per[i] for i in sorted(per)]
    n_per_call = len(ks) // 2 if len(ks) % 2 == 0 else len(ks)
    last = ks[-n_per_call:]
    total = sum(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0) for k in last)
    db = json.load(open(a.out)) if os.path.exists(a.out) else {}
    db[a.workload] = {"bytes_per_launch": total, "replicas": bench.WORKLOADS[a.workload][1],
                      "kernels": {k["kernel"]: k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
                                  for k in last},
                      "source": "ncu dram__bytes_read.sum + dram__bytes_write.sum of one picker_validate_batch "
                                "call over the default shard (scripts/traffic.py, round 2)"}
    json.dump(db, open(a.out, "w"), indent=1)
    print(a.workload, total, [k["kernel"] for k in last])
    sys.exit(0)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_23661_b200 as pk  # noqa: E402

s, rec, args, meta = bench.make_base(a.workload)
p = pk.Picker(0)
p.load(s)
rd, ad = p.replicate(rec, args, meta["ptr_mask"], bench.WORKLOADS[a.workload][1], delta=bench.DELTA)
for _ in range(a.calls):
    p.validate(rd, ad)
torch.cuda.synchronize()
