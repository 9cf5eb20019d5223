# round-2 closing bench lines (after the third-pass captures updated profiles/dram_traffic.json): parity suite,
# per-config bench lines, density cases
mkdir -p gpurun_out/final8
O=gpurun_out/final8
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
for c in 5 1 2 3 4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
for c in 2 5; do timeout 600 python tools/density_case.py --config $c > $O/density_cfg$c.json 2>&1; done
