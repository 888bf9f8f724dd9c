#!/bin/bash
# Same-box A/B of bench configurations: each line "<name>|<bench args>" of $1
# runs bench.py once; one summary line per run (inst/s, frac, parity, kernel ms).
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
while IFS='|' read -r name args; do
  [ -z "$name" ] && continue
  timeout 400 python bench.py $args --no-cpu-baseline --no-latency > gpurun_out/ab_$name.json 2> gpurun_out/ab_$name.err
  python - "$name" "gpurun_out/ab_$name.json" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print("%-28s %8.4g inst/s  frac %.4f  parity %s  call %.4f ms  step %.4f ms" % (sys.argv[1], d["value"], d["roofline"]["frac"], d["parity"]["mismatches"], d["roofline"]["kernel_ms"], d["ms_per_step"]))
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done < "$1"
