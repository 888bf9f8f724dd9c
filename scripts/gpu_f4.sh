# row f4: build, stride tests, f4 row, ncu of the stride module's kernel
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python scripts/rows_bench.py --only f4 --out gpurun_out/rows_f4.json > gpurun_out/rows_f4.log 2>&1
grep -o 'f4_[a-z_]* {"records": [0-9]*, "ms": [0-9.]*\|"frac": [0-9.]*\|"parity_mismatches": [0-9]*\|Error.*' gpurun_out/rows_f4.log | paste -sd' '
timeout 900 python -m pytest tests/test_stride.py -x -q -m gpu > gpurun_out/t_stride.log 2>&1; tail -2 gpurun_out/t_stride.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_validate_pipe -c 1 -o gpurun_out/ncu_f4 python scripts/rows_bench.py --only f4 --steps 1 > gpurun_out/ncu_f4.log 2>&1; tail -1 gpurun_out/ncu_f4.log
