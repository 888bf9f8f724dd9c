# row f1 iteration: build, sequence tests, f1 rows
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_sequence.py -x -q -m gpu > gpurun_out/t_seq.log 2>&1
tail -15 gpurun_out/t_seq.log
timeout 600 python scripts/rows_bench.py --only f1 --out gpurun_out/rows_f1.json > gpurun_out/rows_f1.log 2>&1
tail -5 gpurun_out/rows_f1.log
