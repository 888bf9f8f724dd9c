python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for g in "" "--opt tile=896 --opt threads=448 --opt ctas=2 --opt args_per_rec=5 --opt arg_bufs=1" "--opt tile=768 --opt threads=384 --opt ctas=2 --opt args_per_rec=6 --opt arg_bufs=1" "--opt tile=512 --opt threads=256 --opt ctas=3 --opt args_per_rec=6 --opt arg_bufs=1"; do
  timeout 600 python scripts/rows_bench.py --only f3 --steps 5 $g 2>&1 | grep f3_fused | cut -c1-120 | sed "s|^|[$g] |"
done
