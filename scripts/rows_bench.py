"""The next rows of SURVEY §8 at bench scale, each timed on the device with
CUDA events (median of K steps after W warm-ups) and given an HBM roofline
fraction with the same algorithmic bytes as K1 (32-byte header +
8 bytes per argument per record, + the outputs), against MEASURED_PEAKS.json.

  f1 picker_validate_sequence  C2 x686 (12.5 M records), windows of 32,
                               sequential and concurrent
  f3 picker_consumer_models    C2 x686 with its codes and context sizes (and
     picker_validate_models: verdicts + models in one pass)
  f4 stride-aware K1           C2 x686, module generated stride-aware
  K3 picker_exact_check        C3 small-grid subset x64 (262,144 records)

Verdicts of f1 / K3 are checked against the oracle on the base trace (f1: the
windows of the first replica; K3: a 2,000-record sample).

    python scripts/rows_bench.py [--replicas 686] [--steps 5] [--out profiles/r02_rows.json]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle.picker_oracle as O  # noqa: E402
import paper_2410_23661_b200 as pk  # noqa: E402
from tracegen import workloads  # noqa: E402


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
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--replicas", type=int, default=686)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--out", default=None)
    ap.add_argument("--opt", action="append", default=[], help="library option key=value for the C2 rows (tuning)")
    ap.add_argument("--only", default=None, help="f1 / f3 / f4: only those rows")
    a = ap.parse_args()
    peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6554.6))
    dev = torch.device("cuda", 0)
    out = {"peak_gbs": peak, "rows": {}}

    def row(name, n, nbytes, ms, **kw):
        gbs = nbytes / (ms / 1e3) / 1e9
        out["rows"][name] = {"records": n, "ms": ms, "instances_per_s": n / (ms / 1e3),
                             "algorithmic_bytes": nbytes, "achieved_gbs": gbs, "frac": gbs / peak, **kw}
        print(name, json.dumps(out["rows"][name]), flush=True)

    s, rec, args, meta = workloads.make_c2()
    p = pk.Picker(0, **{k: int(v) for k, v in (o.split("=") for o in a.opt)})
    p.load(s)
    rd, ad = p.replicate(rec, args, meta["ptr_mask"], a.replicas)
    n = rd.shape[0]
    base = 32 * n + 8 * int(ad.numel())
    # f1
    # (default: windows from K1's codes, extents only where no decisive record
    # decides, chosen by the first call; then always from K1's extents)
    for lazy, tag in (((-1, ""), (1, "_lazy"), (0, "_extents")) if a.only in (None, "f1") else ()):
        p.set_option("seq_lazy", lazy)
        for conc in (False, True):
            W = 32
            ms = timed(lambda: p.validate_sequence(rd, ad, W, concurrent=conc), a.steps)
            got = p.validate_sequence(rd[:len(rec)], ad, W, concurrent=conc).cpu().numpy()
            want = np.array(O.oracle_windows(s, rec, args, W, O.SEQ_CONCURRENT if conc else O.SEQ_SEQUENTIAL),
                            np.uint8)
            row(f"f1_windows32_{'concurrent' if conc else 'sequential'}{tag}", n, base + (n + W - 1) // W, ms,
                parity_mismatches=int((got != want).sum()), windows_checked=len(want))
    p.set_option("seq_lazy", -1)
    def run_f4():
        # f4: the stride-aware specialised module
        ps = pk.Picker(0, stride=1)
        ps.load(s)
        fl = torch.empty(n, dtype=torch.uint8, device=dev)
        bt = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
        ct = torch.empty(16, dtype=torch.int64, device=dev)
        ms = timed(lambda: ps.validate(rd, ad, out=(fl, bt, ct)), a.steps)
        got = fl[:len(rec)].cpu().numpy()
        want = np.array(O.oracle_batch_mp(s, rec, args, stride=True), np.uint8)
        row("f4_stride_aware", n, base + n + n / 8, ms, parity_mismatches=int((got != want).sum()))
        ps.close()

    if a.only in ("f1", "f4"):
        if a.only == "f4":
            run_f4()
        if a.out:
            json.dump(out, open(a.out, "w"), indent=1)
        return
    # f3
    flags, _, _ = p.validate(rd, ad)
    ctx = torch.from_numpy((np.arange(n, dtype=np.int64) % 97 + 1) * 4096).to(dev)
    ms = timed(lambda: p.consumer_models(rd, ad, flags, ctx), a.steps)
    row("f3_consumer_models", n, base + n + 8 * n, ms)
    two = p.consumer_models(rd, ad, flags, ctx)
    # f3 fused: verdicts and models in one pass (the K1 bytes + 8 bytes of
    # context size per record); equal to the two passes above
    outs = (torch.empty(n, dtype=torch.uint8, device=dev), torch.empty((n + 31) // 32, dtype=torch.int32, device=dev),
            torch.empty(16, dtype=torch.int64, device=dev))
    ms = timed(lambda: p.validate_models(rd, ad, ctx, out=outs), a.steps)
    (ff, _, _), fused = p.validate_models(rd, ad, ctx, out=outs)
    row("f3_fused_validate_models", n, base + n + n / 8 + 8 * n, ms, launches=p.last_launch_count(),
        equal_to_two_passes=bool(fused == two and torch.equal(ff, flags)))
    p.close()
    if a.only == "f3":
        if a.out:
            json.dump(out, open(a.out, "w"), indent=1)
        return
    run_f4()
    # K3 exact verifier
    s3, r3, a3, m3 = workloads.make_c3(seed=23664, n=4096, n_kernels=32, small=True)
    p3 = pk.Picker(0)
    p3.load(s3)
    rd3, ad3 = p3.replicate(r3, a3, m3["ptr_mask"], 64)
    n3 = rd3.shape[0]
    ms = timed(lambda: p3.exact_check(rd3, ad3), a.steps)
    idx = np.random.default_rng(1).choice(len(r3), 2000, replace=False)
    got = p3.exact_check(rd3[:len(r3)], ad3)[0].cpu().numpy()[idx]
    want = np.array(O.oracle_batch_mp(s3, r3[idx], a3, O.oracle_exact), np.uint8)
    row("K3_exact_c3small_x64", n3, 32 * n3 + 8 * int(ad3.numel()) + n3, ms,
        parity_mismatches=int((got != want).sum()), note="bound by the per-point enumeration, not HBM")
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
