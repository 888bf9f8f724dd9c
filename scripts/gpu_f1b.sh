# row f1 lazy + extents: build, sequence tests, f1 rows
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python scripts/rows_bench.py --only f1 --steps 10 --out gpurun_out/rows_f1.json > gpurun_out/rows_f1.log 2>&1
grep -o 'f1_[a-z0-9_]* {"records": [0-9]*, "ms": [0-9.]*\|"frac": [0-9.]*\|"parity_mismatches": [0-9]*\|Error.*' gpurun_out/rows_f1.log | paste -sd' ' | sed 's/f1_/\nf1_/g'
timeout 1500 python -m pytest tests/test_sequence.py -x -q -m gpu > gpurun_out/t_seq.log 2>&1
tail -15 gpurun_out/t_seq.log
