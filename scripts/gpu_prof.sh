#!/bin/bash
# ncu captures of one workload's main kernel: $1 = workload, $2 = kernel regex, $3 = tag, rest: bench args
w=$1; k=$2; tag=$3; shift 3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/ncu_$tag \
  python bench.py --workload $w --no-cpu-baseline --no-latency --steps 1 --warmup 0 "$@" > gpurun_out/ncu_$tag.log 2>&1
tail -2 gpurun_out/ncu_$tag.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
  python bench.py --workload $w --no-cpu-baseline --no-latency --steps 3 --warmup 1 "$@" > /dev/null 2>&1
tail -12 gpurun_out/launches_$tag.csv
