"""Phase breakdown of one kernel of an ncu report (--set full --import-source):
SASS instructions grouped by how often they executed (per record, per group,
per warp-tile, ...), with their share of instructions and of stall samples,
and the top instructions by stall samples.

    python scripts/ncu_phases.py report.ncu-rep [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
print("#", rows[0][1][:120] if rows and len(rows[0]) > 1 else rep)
hdr = rows[1]
data = rows[2:]
ie = hdr.index("Instructions Executed")
smp = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
vals = [(int(r[ie]) if r[ie].isdigit() else 0, int(r[smp]) if r[smp].isdigit() else 0, r[src].strip()) for r in data]
tot_i = sum(v[0] for v in vals) or 1
tot_s = sum(v[1] for v in vals) or 1
print(f"# {len(vals)} SASS instructions, {tot_i / 1e6:.2f} M warp instructions executed, {tot_s} stall samples")
by = collections.defaultdict(lambda: [0, 0, 0])
for n, s, _ in vals:
    by[n][0] += 1
    by[n][1] += n
    by[n][2] += s
print("\n## by execution count (top 12)")
for n, (c, i, s) in sorted(by.items(), key=lambda x: -x[1][1])[:12]:
    print(f"exec {n:9d} x {c:5d} instr = {i / 1e6:7.2f} M ({100 * i / tot_i:5.1f} % of instructions, "
          f"{100 * s / tot_s:5.1f} % of samples)")
print(f"\n## top {top} instructions by stall samples")
for n, s, t in sorted(vals, key=lambda v: -v[1])[:top]:
    print(f"{s:6d} samples  exec {n:9d}  {t[:90]}")
