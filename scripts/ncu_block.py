"""Print the SASS instructions of one execution-count block of an ncu report
(--set full --import-source) with their stall samples, and an opcode histogram.

    python scripts/ncu_block.py report.ncu-rep EXEC_COUNT [max_lines]
"""
import collections
import csv
import io
import subprocess
import sys

rep, target = sys.argv[1], int(sys.argv[2])
mx = int(sys.argv[3]) if len(sys.argv) > 3 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ie, src, smp = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
sel = [(i, r[src].strip(), r[smp]) for i, r in enumerate(rows[2:]) if r[ie].isdigit() and int(r[ie]) == target]
for i, s, sm in sel[:mx]:
    print(f"{i:6d} {sm:>6s} {s}")
ops = collections.Counter((s.split()[1] if s.startswith("@") else s.split()[0]) for _, s, _ in sel)
print(len(sel), "instructions;", ops.most_common(24))
