# row f3 fused: build, f3 rows, models tests
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python scripts/rows_bench.py --only f3 --out gpurun_out/rows_f3.json > gpurun_out/rows_f3.log 2>&1
grep -o 'f3_[a-z_]* {"records": [0-9]*, "ms": [0-9.]*\|"frac": [0-9.]*\|"equal_to_two_passes": [a-z]*\|Error.*' gpurun_out/rows_f3.log | paste -sd' ' | sed 's/f3_/\nf3_/g'
timeout 900 python -m pytest tests/test_models.py -x -q -m gpu > gpurun_out/t_models.log 2>&1; tail -2 gpurun_out/t_models.log
