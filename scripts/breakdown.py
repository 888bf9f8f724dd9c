"""Row f2: the optimization breakdown of PAPER.md §7.4 (l.1588-1611, Fig. 8b) on
B200 -- Base (per-thread enumeration: picker_exact_check), Base+R (range model,
no range compaction: the summary with every loop descriptor unrolled 32x,
tracegen.uncompact) and Full (range model + compaction: picker_validate_batch).

Workload: the small-grid C3 subset (TVM-style kernels, which "have no unbounded
loops, allowing for effective analysis with our strawman solution", l.1596-1597),
seeded, replicated with pointer relocation for timing.  Each version's verdicts
are checked against the oracle on the base trace (Base: on a sample).

    python scripts/breakdown.py [--replicas R] [--steps K] [--out profiles/r01_breakdown.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2410_23661_b200 as pk  # noqa: E402
from tracegen import workloads  # noqa: E402
from tracegen.uncompact import uncompact  # noqa: E402


def timed(fn, steps, warmup=2):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), float(np.percentile(ts, 90))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--replicas", type=int, default=64)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--unroll", type=int, default=32)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    s, rec, args, meta = workloads.make_c3(seed=23664, n=4096, n_kernels=32, small=True)
    su = uncompact(s, a.unroll)
    rr, aa = workloads.replicate(rec, args, meta["ptr_mask"], a.replicas)
    n = len(rr)
    dev = torch.device("cuda", 0)
    rec_d = torch.from_numpy(rr.view(np.uint8).reshape(-1, 32)).to(dev)
    args_d = torch.from_numpy(aa).to(dev)
    flags = torch.empty(n, dtype=torch.uint8, device=dev)
    bits = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
    counts = torch.empty(16, dtype=torch.int64, device=dev)

    full = pk.Picker(0)
    full.load(s)
    base_r = pk.Picker(0)
    base_r.load(su)
    out = {"workload": f"C3 small-grid subset (seed 23664, 4096 records, 32 kernels) x{a.replicas}",
           "records": n, "unroll": a.unroll,
           "descriptors_per_kernel": {
               "full": float(np.mean([len(k["desc"]) for k in s["kernels"]])),
               "base_r": float(np.mean([len(k["desc"]) for k in su["kernels"]]))}}
    res = {}
    for name, p in (("full", full), ("base_r", base_r)):
        ms, p90 = timed(lambda p=p: p.validate(rec_d, args_d, out=(flags, bits, counts)), a.steps)
        res[name] = {"ms_per_batch": ms, "ms_p90": p90, "instances_per_s": n / (ms / 1e3),
                     "us_per_instance": 1e3 * ms / n}
        res[name]["codes"] = flags[:len(rec)].cpu().numpy()
    # Base: the exact verifier (synchronous call; fewer records -- it enumerates)
    nb = min(n, 8 * len(rec))
    ex = pk.Picker(0)
    ex.load(s)
    t0 = time.perf_counter()
    codes_b, _ = ex.exact_check(rec_d[:nb], args_d, max_points=1 << 24)
    torch.cuda.synchronize()
    ms_b, p90_b = timed(lambda: ex.exact_check(rec_d[:nb], args_d, max_points=1 << 24), max(3, a.steps // 3), 1)
    res["base"] = {"ms_per_batch": ms_b, "ms_p90": p90_b, "records": nb, "instances_per_s": nb / (ms_b / 1e3),
                   "us_per_instance": 1e3 * ms_b / nb, "codes": codes_b[:len(rec)].cpu().numpy()}
    # parity with the oracle (test infrastructure) on the base trace
    import oracle.picker_oracle as O
    want_f = np.array(O.oracle_batch_mp(s, rec, args), np.uint8)
    want_u = np.array(O.oracle_batch_mp(su, rec, args), np.uint8)
    idx = np.random.default_rng(0).choice(len(rec), 256, replace=False)
    want_e = np.array(O.oracle_batch_mp(s, rec[idx], args, O.oracle_exact, cap=1 << 24), np.uint8)
    parity = {"full": int((res["full"]["codes"] != want_f).sum()),
              "base_r": int((res["base_r"]["codes"] != want_u).sum()),
              "base_sample256": int((res["base"]["codes"][idx] != want_e).sum())}
    # range-overestimation conservatism, measured by the
    # exact verifier: interval NI (10) where the exact byte sets are disjoint (0);
    # and how many of those the stride-aware variant (row f4) recovers
    full_c, base_c = res["full"]["codes"], res["base"]["codes"]
    st = pk.Picker(0)
    st.set_option("stride", 1)
    st.load(s)
    stride_c, _, _ = st.validate(rec, args)
    stride_c = stride_c.cpu().numpy()
    ro = (full_c == 10) & (base_c == 0)
    out["ro_conservatism"] = {"records": int(len(rec)), "interval_ni": int((full_c == 10).sum()),
                              "exact_ni": int((base_c == 10).sum()), "interval_ni_exact_i": int(ro.sum()),
                              "recovered_by_stride": int((ro & (stride_c == 0)).sum()),
                              "stride_unsound": int(((base_c == 10) & (stride_c == 0)).sum())}
    for v in res.values():
        c = v.pop("codes")
        v["verdicts"] = {int(k): int(x) for k, x in zip(*np.unique(c, return_counts=True))}
    out["versions"] = res
    out["parity_mismatches"] = parity
    out["speedup"] = {"full_vs_base_r": res["full"]["instances_per_s"] / res["base_r"]["instances_per_s"],
                      "full_vs_base": res["full"]["instances_per_s"] / res["base"]["instances_per_s"]}
    line = json.dumps(out)
    print(line)
    if a.out:
        with open(a.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
