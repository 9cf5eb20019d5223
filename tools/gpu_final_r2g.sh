# round-2 closing lines after the fill's per-round prefix packs: parity suite, smoke, bench lines cfg 1-5,
# density / symmetric / tree-order cases
mkdir -p gpurun_out/final11
O=gpurun_out/final11
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
for c in 5 1 2 3 4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
for c in 2 5; do
  timeout 600 python tools/density_case.py --config $c > $O/density_cfg$c.json 2>&1
  timeout 300 python tools/run_case.py --config $c --reps 3 --symmetric > $O/sym_cfg$c.json 2>&1
  timeout 300 python tools/run_case.py --config $c --reps 3 --tree-order > $O/tree_order_cfg$c.json 2>&1
done
tail -3 $O/gpu_tests.log; tail -1 $O/smoke.log
