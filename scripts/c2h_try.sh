# C2-heavy: schedule / option experiments (same box)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for o in "" "--opt sorted=1" "--opt loop_min=4" "--opt loop_min=3"; do
  timeout 300 python bench.py --workload c2heavy --no-cpu-baseline --no-latency --steps 10 $o > gpurun_out/c2h.json 2> gpurun_out/c2h.err
  python - "$o" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/c2h.json").read().strip().splitlines()[-1])
    print(repr(sys.argv[1]), "%.4g inst/s" % d["value"], "frac %.4f" % d["roofline"]["frac"], "parity", d["parity"]["mismatches"])
except Exception as e:
    print(sys.argv[1], "FAILED", e, open("gpurun_out/c2h.err").read()[-300:])
PY
done
