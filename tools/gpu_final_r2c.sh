# round-2 closing evidence (third pass, final: shared-memory staging, per-warp arena bounds,
# symmetric thresholds in the test block, exact band by candidate, unit preparation in the
# descent): parity suite, per-config bench lines, launch lists, ncu --set full of the search kernels (cfg 5 and 2), density / symmetric / tree-order cases
mkdir -p gpurun_out/final7
O=gpurun_out/final7
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
for c in 5 1 2 3 4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_cfg5.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-tree-order > $O/ncu_launch.log 2>&1
for c in 2 3 4; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_cfg$c.csv python tools/run_case.py --config $c --reps 1 > $O/ncu_launch_cfg$c.log 2>&1
done
timeout 1800 ncu --set full --import-source on --clock-control none -k regex:"walk_kernel|fill_kernel|desc_kernel" -c 3 \
  -o $O/k_full -f python tools/run_case.py --config 5 --reps 1 > $O/ncu_k.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"walk_kernel|fill_kernel|desc_kernel" -c 3 \
  -o $O/k2_full -f python tools/run_case.py --config 2 --reps 1 > $O/ncu_k2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fill_kernel" -c 1 \
  -o $O/fill_to -f python tools/run_case.py --config 5 --reps 1 --tree-order > $O/ncu_fill_to.log 2>&1
for c in 2 5; do
  timeout 600 python tools/density_case.py --config $c > $O/density_cfg$c.json 2>&1
  timeout 300 python tools/run_case.py --config $c --reps 3 --symmetric > $O/sym_cfg$c.json 2>&1
  timeout 300 python tools/run_case.py --config $c --reps 3 --tree-order > $O/tree_order_cfg$c.json 2>&1
done
