#!/bin/bash
# Every bench workload once (1 GPU), one JSON line each, into gpurun_out/$1_bench_<workload>.json
tag=${1:-r02}
for w in c2 c2r1 c2heavy c3 c4 wide; do
  extra="--no-cpu-baseline --no-latency"
  [ "$w" = "c2" ] && extra=""
  timeout 400 python bench.py --workload $w $extra > gpurun_out/${tag}_bench_$w.json 2> gpurun_out/${tag}_bench_$w.err
  python - "$w" "gpurun_out/${tag}_bench_$w.json" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], "%.3g inst/s" % d["value"], "frac %.3f" % d["roofline"]["frac"], "parity", d["parity"]["mismatches"], "ms", round(d["ms_per_step"], 4))
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
