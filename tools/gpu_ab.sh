# A/B timing of library variants (paper_1910_02639_b200/libbtree_*.so), interleaved twice, per-rep phases; clocks sampled
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.mem,temperature.gpu,power.draw,clocks_throttle_reasons.active --format=csv -lms 500 > gpurun_out/ab_clocks.csv 2>&1 &
SMI=$!
for r in 1 2; do
  for f in paper_1910_02639_b200/libbtree_*.so; do
    v=$(basename $f .so)
    BT_LIB=$PWD/$f timeout 300 python tools/run_case.py --config ${1:-5} --reps 4 ${2:-} > gpurun_out/ab_${v}_r$r.json 2>&1
  done
done
kill $SMI
