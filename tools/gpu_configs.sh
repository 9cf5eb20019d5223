# per-config bench lines (BASELINE.json configs 1..5) + the full oracle baselines, on one B200 box
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r02_bench_cfg$c.json 2> gpurun_out/r02_bench_cfg$c.err
done
timeout 2400 python tools/oracle_baseline.py --configs 1 2 3 4 5 --single 1 2 3 4 > gpurun_out/r02_oracle_baseline.jsonl 2> gpurun_out/r02_oracle_baseline.err
