python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for g in "" "--opt tile=768 --opt threads=384 --opt ctas=2 --opt args_per_rec=5 --opt arg_bufs=1" "--opt tile=640 --opt threads=320 --opt ctas=2 --opt args_per_rec=6 --opt arg_bufs=1" "--opt tile=1024 --opt threads=256 --opt ctas=2 --opt args_per_rec=5 --opt arg_bufs=1"; do
  timeout 600 python scripts/rows_bench.py --only f3 --steps 5 $g 2>&1 | grep f3_fused | cut -c1-200 | sed "s|^|[$g] |"
done
