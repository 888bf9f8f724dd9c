"""Row f3: the paper's two case studies (§7.5 l.1612-1690) as analytic
models evaluated on the device over the C2 trace's verdicts
(picker_consumer_models): Asymmetric-Resilience checkpoint bytes and Chimera
preemption latency, per application and in total.

Context sizes (synthetic; recipe in DESIGN.md §8): log-linear in the
instance's resident threads, scaled so a save takes 4 us (one warp) to 98 us
(a full GPU) at 1,000 bytes/us -- the paper's band (l.1683-1684).  Kill latency 1 us
(l.1677-1679).  Also times the model pass on the full bench trace.

    python scripts/case_studies.py [--out profiles/r01_case_studies.json]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2410_23661_b200 as pk  # noqa: E402
from tracegen import workloads  # noqa: E402

SAVE_BPU = 1000


def context_bytes(rec):
    """Synthetic saved-context size: log-linear in the instance's resident
    threads (min(threads, 148 SMs x 2048)), scaled so that at SAVE_BPU bytes/us
    a save takes 4 us (32 threads) to 98 us (a full GPU) -- the paper's band."""
    thr = (rec["grid_x"].astype(np.int64) * rec["grid_y"] * rec["grid_z"]
           * rec["block_x"] * rec["block_y"] * rec["block_z"])
    lo, hi = 5.0, np.log2(148 * 2048)
    t = (np.clip(np.log2(np.maximum(thr, 1)), lo, hi) - lo) / (hi - lo)
    return np.round((4.0 + 94.0 * t) * SAVE_BPU).astype(np.uint64)


def summarize(m):
    n = max(m["n"], 1)
    return {"n": m["n"], "idempotent": m["n_idem"],
            "ar_ckpt_bytes_without": m["ckpt_bytes_all"], "ar_ckpt_bytes_with": m["ckpt_bytes_ni"],
            "ar_bytes_saved_pct": 100.0 * (1 - m["ckpt_bytes_ni"] / max(m["ckpt_bytes_all"], 1)),
            "unknown_input": m["unknown_input"],
            "chimera_mean_us_without": m["preempt_ns_without"] / n / 1e3,
            "chimera_mean_us_with": m["preempt_ns_with"] / n / 1e3,
            "chimera_reduction_pct": 100.0 * (1 - m["preempt_ns_with"] / max(m["preempt_ns_without"], 1)),
            "chimera_within_1us_pct": 100.0 * (m["hist_with"][0] + m["hist_with"][1]) / n}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--replicas", type=int, default=686)
    a = ap.parse_args()
    s, rec, args, meta = workloads.make_c2()
    p = pk.Picker(0)
    p.load(s)
    flags, _, _ = p.validate(rec, args)
    ctx = context_bytes(rec)
    out = {"workload": "C2 trace (547 kernels / 18,217 instances / 6 apps)", "save_bytes_per_us": SAVE_BPU,
           "kill_ns": 1000, "apps": {}}
    out["all"] = summarize(p.consumer_models(rec, args, flags, ctx, save_bytes_per_us=SAVE_BPU))
    for i, name in enumerate(meta["apps"]):
        sel = np.nonzero(meta["app"] == i)[0]
        if len(sel) == 0:
            continue
        m = p.consumer_models(rec[sel], args, flags[torch.from_numpy(sel).to(flags.device)], ctx[sel],
                              save_bytes_per_us=SAVE_BPU)
        out["apps"][name] = summarize(m)
    # time the fused model pass on the bench trace (device-resident)
    rr, aa = workloads.replicate(rec, args, meta["ptr_mask"], a.replicas)
    dev = torch.device("cuda", 0)
    rd = torch.from_numpy(rr.view(np.uint8).reshape(-1, 32)).to(dev)
    ad = torch.from_numpy(aa).to(dev)
    fl, _, _ = p.validate(rd, ad)
    cd = torch.from_numpy(np.tile(ctx, a.replicas).view(np.int64)).to(dev)
    p.consumer_models(rd, ad, fl, cd, save_bytes_per_us=SAVE_BPU)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        p.consumer_models(rd, ad, fl, cd, save_bytes_per_us=SAVE_BPU)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out["model_pass"] = {"records": len(rr), "ms": float(np.median(ts)),
                         "instances_per_s": len(rr) / (float(np.median(ts)) / 1e3)}
    line = json.dumps(out)
    print(line)
    if a.out:
        open(a.out, "w").write(line + "\n")


if __name__ == "__main__":
    main()
