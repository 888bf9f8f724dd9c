"""Write the specialised-module source generated for a bench workload to
picker_jit.cu (the file name NVRTC records in the line table), so that
`ncu --import-source on` can attach it to the profile."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_23661_b200.validator import compile_summaries  # noqa: E402
from tracegen import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--out", default="picker_jit.cu")
a = ap.parse_args()
if a.workload == "c2":
    summary = workloads.make_c2()[0]
elif a.workload == "c3":
    summary = workloads.make_c3()[0]
else:
    summary = workloads.make_c4()[0]
r, msg, src = compile_summaries(summary, want_source=True)
open(a.out, "w").write(src)
print(r, msg[:120])
