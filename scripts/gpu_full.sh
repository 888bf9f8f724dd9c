#!/bin/bash
# Full GPU suite + the A/B bench list (scripts/ab_list.txt) on one box.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
tail -4 gpurun_out/gpu_tests.log
bash scripts/ab_bench.sh scripts/ab_list.txt
