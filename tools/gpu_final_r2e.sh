# round-2 closing check after the fill store policy: parity suite, smoke, bench lines cfg 5 and 2
mkdir -p gpurun_out/final9
O=gpurun_out/final9
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
for c in 5 2; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
