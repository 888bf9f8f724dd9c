#!/bin/bash
# A/B harness for kernel experiments on one GPU box.
#   scripts/ab.sh NAME[:PATCH] ...     (no PATCH: the tree as it is)
# Each variant is a copy of the repo under /tmp/ab_NAME with PATCH applied
# (patch -p1), built in its copy, then timed on C2 / C3 / C4 (bench.py,
# parity checked, no latency / e2e / CPU legs).  One summary line per run is
# appended to gpurun_out/ab.txt.  WORKLOADS overrides the workload list.
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/gpurun_out
mkdir -p "$OUT"
WL=${WORKLOADS:-"c2 c3 c4"}
for spec in "$@"; do
  name=${spec%%:*}
  patch=""
  [[ "$spec" == *:* ]] && patch=${spec#*:}
  dir=/tmp/ab_$name
  rm -rf "$dir" /tmp/ab_cache_$name
  mkdir -p "$dir"
  (cd "$ROOT" && tar --exclude=./gpurun_out --exclude=./.git -cf - .) | (cd "$dir" && tar xf -)
  if [ -n "$patch" ]; then
    (cd "$dir" && patch -p1 -s < "$ROOT/$patch") || { echo "$name: patch failed" >> "$OUT/ab.txt"; continue; }
  fi
  (cd "$dir" && python -c "import __graft_entry__ as g; g.build()") > "$OUT/ab_build_$name.log" 2>&1 ||
    { echo "$name: build failed" >> "$OUT/ab.txt"; continue; }
  for w in $WL; do
    # a JIT module cache of its own per variant (variants can share generated source)
    (cd "$dir" && PICKER_JIT_CACHE=/tmp/ab_cache_$name timeout 300 python bench.py --workload "$w" --steps 20 --warmup 5 --no-cpu-baseline \
       --no-latency --e2e-steps 1 ${AB_OPTS:-}) > "$OUT/ab_${name}_$w.json" 2> "$OUT/ab_${name}_$w.err"
    python - "$OUT/ab_${name}_$w.json" "$name" "$w" >> "$OUT/ab.txt" <<'EOF'
import json, sys
path, name, w = sys.argv[1:]
try:
    d = json.loads(open(path).read().strip().splitlines()[-1])
    print(f"{name:12s} {w}: {d['value']/1e9:8.3f} G inst/s  kernel {d['roofline']['kernel_ms']:.4f} ms  "
          f"frac {d['roofline']['frac']:.3f}  mismatches {d['parity']['mismatches']}  sm {d['clocks']['sm_mhz']}")
except Exception as e:  # noqa: BLE001
    print(f"{name:12s} {w}: FAILED ({e})")
EOF
  done
done
