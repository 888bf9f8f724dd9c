#!/bin/bash
# Round-end evidence on one GPU: smoke, the default bench line (+ reference arm),
# every workload, the rows, the launch list of the default bench command and a
# full ncu capture of its dominant kernel.  Outputs under gpurun_out/ (tag $1).
tag=${1:-r02}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; tail -1 gpurun_out/${tag}_smoke.log
timeout 600 python bench.py > gpurun_out/${tag}_bench_c2.json 2> gpurun_out/${tag}_bench_c2.err; tail -c 300 gpurun_out/${tag}_bench_c2.json
timeout 600 python bench.py --impl reference > gpurun_out/${tag}_bench_reference.json 2> gpurun_out/${tag}_bench_reference.err
for w in c2r1 c2heavy c3 c4 wide; do
  timeout 400 python bench.py --workload $w --no-cpu-baseline --no-latency > gpurun_out/${tag}_bench_$w.json 2> gpurun_out/${tag}_bench_$w.err
done
timeout 1200 python scripts/rows_bench.py --out gpurun_out/${tag}_rows.json > gpurun_out/${tag}_rows.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_c2.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-latency > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_validate_pipe -c 1 -o gpurun_out/${tag}_ncu_c2 \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-latency > gpurun_out/${tag}_ncu_c2.log 2>&1
for w in c2r1 c2heavy c3 c4 wide; do
  python - "$w" "gpurun_out/${tag}_bench_$w.json" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], "%.4g inst/s" % d["value"], "frac %.4f" % d["roofline"]["frac"], "parity", d["parity"]["mismatches"])
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
