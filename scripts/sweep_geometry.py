"""Sweep the specialised kernel's geometry (tile, threads, CTAs/SM) on the bench
workload; prints instances/s per setting (tuning aid, not a bench line)."""
import itertools
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_23661_b200 as pk  # noqa: E402
from tracegen.workloads import make_c2, make_c3, make_c4, replicate  # noqa: E402


def main():
    w = os.environ.get("WORKLOAD", "c2")
    reps = int(os.environ.get("REPLICAS", {"c2": "686", "c3": "64", "c4": "512"}[w]))
    s, rec, a, meta = {"c2": make_c2, "c3": lambda: make_c3(n=1 << 14, n_kernels=64),
                       "c4": lambda: make_c4(n=1 << 13, n_kernels=32)}[w]()
    R, A = replicate(rec, a, meta["ptr_mask"], reps, 1 << 37)
    dev = torch.device("cuda", 0)
    rd = torch.from_numpy(R.view(np.uint8).reshape(-1, 32)).to(dev)
    ad = torch.from_numpy(A).to(dev)
    n = len(R)
    flags = torch.empty(n, dtype=torch.uint8, device=dev)
    bits = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
    cnt = torch.empty(16, dtype=torch.int64, device=dev)
    ref = None
    cfgs = os.environ.get("CONFIGS", "512/256/2/8")
    for cfg in cfgs.split(","):
        t, th, c, apr = (int(x) for x in cfg.split("/"))
        try:
            p = pk.Picker(0, tile=t, threads=th, ctas=c, args_per_rec=apr)
            p.load(s)
        except Exception as e:  # noqa: BLE001
            print(f"{cfg}: {str(e)[:100]}")
            continue
        for _ in range(3):
            p.validate(rd, ad, out=(flags, bits, cnt))
        torch.cuda.synchronize()
        if ref is None:
            ref = flags.clone()
        ok = bool(torch.equal(flags, ref))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            p.validate(rd, ad, out=(flags, bits, cnt))
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"tile={t:5d} threads={th:4d} ctas={c} apr={apr}: {ms:7.3f} ms  {n / ms / 1e6:7.2f} G inst/s  "
              f"same={ok}", flush=True)
        p.close()


if __name__ == "__main__":
    main()
