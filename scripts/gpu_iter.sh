set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_wide.py -x -q > gpurun_out/t_wide.log 2>&1
tail -3 gpurun_out/t_wide.log
timeout 400 python bench.py --workload wide --no-cpu-baseline --no-latency > gpurun_out/b_wide.json 2> gpurun_out/b_wide.err
tail -c 1500 gpurun_out/b_wide.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_validate_wide -c 1 -o gpurun_out/ncu_wide python bench.py --workload wide --no-cpu-baseline --no-latency --steps 1 --warmup 0 > gpurun_out/ncu_wide.log 2>&1
tail -3 gpurun_out/ncu_wide.log
