# ncu capture of the fused f1 kernel (second call of scripts/f1_once.py)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python scripts/f1_once.py > gpurun_out/f1_once.log 2>&1; tail -2 gpurun_out/f1_once.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_validate_pipe --launch-skip 1 -c 1 -o gpurun_out/ncu_f1 python scripts/f1_once.py > gpurun_out/ncu_f1.log 2>&1
tail -2 gpurun_out/ncu_f1.log
