# f1 fused: geometry sweep of the extents module (tile threads ctas apr bufs)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for g in "448 448 2 5 1" "448 224 2 5 1" "896 448 1 5 2" "448 224 2 5 2" "672 224 1 5 2"; do
  set -- $g
  echo "== $g"
  timeout 300 python scripts/rows_bench.py --only f1 --opt tile=$1 --opt threads=$2 --opt ctas=$3 --opt args_per_rec=$4 --opt arg_bufs=$5 2>&1 | grep -o '"ms": [0-9.]*\|f1_windows32_[a-z]*\|Error.*' | paste -sd' '
done
